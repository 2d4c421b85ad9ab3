// detector.cpp -- the B200 step driver: one data-parallel Faster R-CNN ResNet-C4
// training step as a static C++ schedule over the sm_100a kernels.
//
// Mirrors the reference step body (src/trainer.cpp:217-271, order in
// SURVEY.md Appendix B):
//   fp16 shadows of conv/fc weights, BN params fp32      trainer.cpp:222-227
//   forward (every fp16 op output rounded RNE)            tensor.cpp:79-82
//   losses with the loss scale folded into backward      model.cpp:132-150
//   backward, grads finalised in the leaf dtype           autograd.cpp:437-485
//   loss allreduce /K; gradient allreduce (fp16 buckets,  trainer.cpp:240-251
//     issued as each bucket's last wgrad completes, overlapped with backward)
//   overflow = nonfinite(summed grads); fused unscale+SGD trainer.cpp:252-254,86-94
//   update_scale                                          precision.cpp:45-56
// The reference's Tape/CustomOp machinery (autograd.cpp) is replaced by this
// fixed schedule; all activations live in HBM buffers allocated once, and the
// whole step is captured into a CUDA graph after the first (eager) step.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <nvtx3/nvToolsExt.h>
#include <fstream>
#include <stdexcept>
#include <string>
#include <map>
#include <vector>

#include "../../include/sdb.h"
#include "ctx.h"
#include "detect.h"
#include "sdb_internal.h"

using namespace sdb;

namespace {

int det_fail(int code, const std::string& m) { return sdb::set_error(code, m.c_str()); }

// a failed NCCL call (its message is in sdb_last_error): maps to SDB_COLLECTIVE
struct CollectiveFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
#define CKC(expr)                                                                         \
    do {                                                                                  \
        if ((expr) != cudaSuccess) throw CollectiveFailure(std::string(#expr) + ": " + sdb_last_error()); \
    } while (0)

#define CK(expr)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess) throw std::runtime_error(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

uint64_t mix64(uint64_t a, uint64_t b) {
    uint64_t z = a ^ (b + 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// splitmix64 Rng of the reference (src/tensor.cpp:38-49), for bit-identical init
struct Rng {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    float uniform(float lo, float hi) {
        const float u = static_cast<float>(next() >> 40) * 0x1.0p-24f;
        return lo + (hi - lo) * u;
    }
};

int round_up(int v, int m) { return (v + m - 1) / m * m; }

struct Act {
    void* p = nullptr;
    int n = 0, h = 0, w = 0, c = 0;
    int64_t numel() const { return static_cast<int64_t>(n) * h * w * c; }
};

struct Param {
    std::string name;
    std::vector<int64_t> ref_shape;
    int kind = 0;  // 0 conv, 1 fc, 2 gamma, 3 beta
    int64_t off = 0, numel = 0;  // in the conv/fc flat or the bn flat
    int K = 0, R = 1, S = 1, C = 0;  // device KRSC dims (conv/fc)
};

struct ConvL {
    int p = -1;  // param index
    ConvShape g{};
};

struct NormL {
    int pg = -1, pb = -1;  // gamma/beta param index
    int C = 0;
    float* mean = nullptr;
    float* invstd = nullptr;
    float* agg = nullptr;  // sync_bn: [sum, sumsq, count] of the forward, summed over ranks
    int act = 0;  // mode 0: 0 none / 1 relu; mode 1: 2 (iabn)
    float slope = 1.0f;
};

struct Block {
    ConvL c1, c2, c3, down;
    NormL n1, n2, n3, nd;
    bool has_down = false;
    Act in, z1, a1, z2, a2, z3, b3, zd, d, out;
    // sign bitmap of `out` ([rows][C/8] bytes, bit = out > 0), written by the
    // fused bn3 apply (IABN fp16) for the next layer's dgrad-epilogue mask
    uint8_t* obits = nullptr;
};

enum ProfCat {
    P_FPROP = 0, P_DGRAD, P_WGRAD, P_NORM_F, P_NORM_B, P_ELEM, P_POOL, P_TARGETS, P_PROPOSAL, P_ROI_F, P_ROI_B,
    P_LOSS, P_OPTIM, P_COMM, P_NCAT
};

// per-category CUDA-event timing of one eager step (sdb_det_profile)
struct Prof {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> recs;
    std::vector<std::string> labels;
    std::vector<double> rec_flops, rec_bytes;
    double flops[P_NCAT] = {}, bytes[P_NCAT] = {};
    int64_t launches[P_NCAT] = {};
    struct Rec {
        int cat;
        std::string label;
        double ms, flops, bytes;
    };
    std::vector<Rec> last;  // the last profiled step, per labelled record
    cudaEvent_t get() {
        if (used == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        return pool[used++];
    }
};

}  // namespace

struct sdb_det {
    sdb_ctx* ctx = nullptr;
    sdb_det_config cfg{};
    int dt = kF16;
    int es = 2;
    std::vector<Param> params;
    int64_t n_w = 0, n_bn = 0;
    // flat parameter state
    float *w32 = nullptr, *v32 = nullptr, *bn32 = nullptr, *bnv = nullptr, *bng = nullptr;
    void* wdev = nullptr;  // weights used by the kernels: fp16 shadow (mode 1) or w32 (mode 0)
    void* g = nullptr;     // conv/fc grads (dtype)
    // loss-scale state + outputs
    double* scale = nullptr;
    int64_t* good = nullptr;
    int* flag = nullptr;
    double* losses = nullptr;      // [8]: 4 losses, (reduced copy)
    double* scale_used = nullptr;  // snapshot of the scale used by the step
    // layers
    ConvL stem;
    NormL stem_n;
    Act img, stem_z, stem_a, pool;
    // fp16: the stem as a 1x1 GEMM over its im2col matrix (stem2.g = [1][1][pixels][192] -> 64)
    bool stem_gemm = false;
    ConvL stem2;
    void *stem_x2 = nullptr, *stem_w2 = nullptr, *stem_dw2 = nullptr;
    uint8_t* pool_arg = nullptr;
    std::vector<Block> backbone, head;
    // sqrt(L) activation checkpointing of the backbone blocks (memory.checkpoint,
    // src/memopt.cpp:76-89 plan, :150-210 runner): ck_start = segment starts + L;
    // every tensor of a segment except its last block's output lives in one
    // arena shared by all segments, refilled by a forward recompute in backward
    std::vector<int> ck_start;
    uint8_t* ck_arena = nullptr;
    size_t ck_off = 0, ck_bytes = 0;
    bool measuring = false;        // sizing pass: no device allocation
    cudaEvent_t ck_ev = nullptr;   // side-stream wgrads done with an arena segment
    int64_t bytes_total = 0, bytes_backbone = 0;
    ConvL rpn_conv, rpn_cls, rpn_bbox, fc_cls, fc_bbox;
    Act c4, rpn_z, rpn_a, rpn_logits, rpn_deltas, roi_feat, head_out, pooled, cls_logits, bbox_pred;
    int A = 0, A_pad = 0, n_loc = 0, nA = 0, fh = 0, fw = 0, ncls = 0, ncls_pad = 0, nbox_pad = 0;
    int R = 0, P = 0, head_hw = 0, feat_c = 0;
    int roi_step = 1;  // RoIAlign bin subsampling folded from a 1x1 stride-2 head entry
    // deferred split-K wgrad reduction (fp16): every conv keeps its fp32
    // partials in its own arena slice; each gradient bucket is reduced by one
    // batched launch as soon as the last wgrad of the bucket has been issued
    // (then, with a communicator, allreduced) -- the same schedule at every
    // world size
    bool defer_wgrad = false;
    uint8_t* wg_arena = nullptr;
    std::map<int, size_t> wg_off;  // param index -> arena byte offset
    struct BucketTab {
        WgradJob* jobs = nullptr;  // device job table (uploaded at the first step)
        int* tiles = nullptr;      // tile prefix of the jobs
        int njobs = 0, total = 0;
    };
    std::vector<int> bucket_of;                // param index -> bucket (conv/fc), -1 otherwise
    std::vector<int> bucket_nparams;           // conv/fc params per bucket
    std::vector<int> bucket_left;              // this step: params whose wgrad is not issued yet
    std::vector<std::vector<WgradJob>> bjobs;  // this step: issued jobs per bucket
    std::vector<BucketTab> btab;
    // the deferred wgrads run on a side stream, overlapping the dgrad -> norm
    // backward chain; each takes its dz from a ring whose slots are recycled
    // only after the wgrad that read them has finished
    static constexpr int kDzRing = 64;  // capacity; dzr_n slots in use
    int dzr_n = 6;
    bool side_wgrad = false;
    // the last RoI-head block's output is average-pooled inside its apply pass
    // and never stored (only its sign bitmap); head_out is then not materialised
    bool head_pool_fuse = false;
    const void* dpool_cur = nullptr;  // this step's pooled gradient (head_pool_fuse)
    bool head_pool_bwd = false;       // the last block's bn3 backward forms the pool gradient itself
    cudaStream_t wst = nullptr;
    cudaEvent_t wev_fork = nullptr, wev_join = nullptr;
    void* dzr[kDzRing] = {};
    // anchor targets depend only on the fed GT: they run on the side stream
    // at the start of the step, behind the backbone forward
    void* ws_at = nullptr;
    cudaEvent_t ev_at_fork = nullptr, ev_at_join = nullptr;
    // the RPN losses and RPN head backward (all but the rpn_conv dgrad, which
    // accumulates onto the RoIAlign gradient) also run there, while the main
    // stream is in the latency-bound proposal layer and the RoI head
    cudaEvent_t ev_rpn_fork = nullptr, ev_rpn_join = nullptr;
    // the downsampling shortcut (down conv + its norm) of a stage's first block
    // runs on bst, concurrently with the block's conv1-conv3 chain (forward)
    cudaStream_t bst = nullptr;
    cudaEvent_t ev_b_fork = nullptr, ev_b_join = nullptr;
    ConvStats cst2{};
    // backward twin: the shortcut's norm backward + dgrad on bst (dz into dzb,
    // whose wgrad on the side stream must finish before the next reuse: ev_dzb)
    void* dzb = nullptr;
    cudaEvent_t ev_b2_fork = nullptr, ev_dzb = nullptr;
    bool dzb_busy = false;
    void* drpn_side = nullptr;
    cudaEvent_t dzr_ev[kDzRing] = {};
    bool dzr_busy[kDzRing] = {};
    int dzr_next = 0;
    void* img3 = nullptr;  // device staging of [N][3][H][W] host images (train_step_host_nchw)
    float* anchors = nullptr;
    // targets
    float* gt = nullptr;
    int32_t *gt_cls = nullptr, *gt_count = nullptr;
    uint64_t* keys = nullptr;  // [2*batch]: rpn keys then rcnn keys
    int8_t* a_labels = nullptr;
    float* a_targets = nullptr;
    float* props = nullptr;
    int32_t *prop_count = nullptr, *keep_pos = nullptr;
    int8_t* pt_flag = nullptr;
    int32_t* pt_arg = nullptr;
    float* rois = nullptr;
    int32_t *roi_labels = nullptr, *roi_count = nullptr;
    float* roi_targets = nullptr;
    // grad scratch
    void* gbuf[5] = {};
    void *d_rpn_logits = nullptr, *d_rpn_deltas = nullptr, *d_cls = nullptr, *d_bbox = nullptr;
    int64_t gbuf_elems = 0;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    // fused output statistics of the fprop that precedes each norm layer
    ConvStats cst{};
    // fused InPlace-ABN backward statistics of the dgrad that produces a norm
    // layer's output gradient (bn1 / bn2 of every bottleneck)
    ConvStats cst_b{};
    // host staging, double-buffered: a call waits only for the copies that
    // read its slot two calls ago (never for the previous step's compute)
    static constexpr int kStage = 2;
    float* h_gt[kStage] = {};
    int32_t *h_cls[kStage] = {}, *h_cnt[kStage] = {};
    uint64_t* h_keys[kStage] = {};
    int64_t* h_slots[kStage] = {};
    cudaEvent_t stage_ev[kStage] = {};
    bool stage_busy[kStage] = {};
    int stage_next = 0;
    int64_t* slots_dev = nullptr;
    double* h_losses = nullptr;
    // comm: an NCCL communicator exists (world > 1, or a forced 1-rank one that
    // runs the data-parallel code path on one GPU)
    bool comm_on = false;
    float* sbn_red = nullptr;  // sync_bn backward sums [2 * max C]
    void* ws2 = nullptr;       // workspace of the concurrent shortcut branch
    // sharded optimizer: buckets are reduce-scattered, each rank
    // updates its 1/K shard of the fp32 masters and all-gathers the fp16 shadows
    bool shard = false;
    bool masters_synced = true;  // the full fp32 masters are current on this rank
    std::vector<cudaEvent_t> gather_ev;
    cudaEvent_t ev_gather_join = nullptr;
    cudaStream_t comm = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::vector<cudaEvent_t> bucket_ev;
    std::vector<std::pair<int64_t, int64_t>> buckets;  // [lo, hi) element ranges of g, issued from the end
    // graph
    cudaGraphExec_t gexec = nullptr;
    bool use_graph = true;
    int steps_done = 0;
    int64_t launches = 0;
    std::vector<void*> allocs;
    Prof prof;

    void* alloc(size_t bytes) {
        if (measuring) return nullptr;
        void* p = nullptr;
        CK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
        allocs.push_back(p);
        bytes_total += static_cast<int64_t>(std::max<size_t>(bytes, 256));
        return p;
    }
    // a slice of the checkpoint arena (256-byte aligned)
    void* seg_alloc(size_t bytes) {
        const size_t off = ck_off;
        ck_off += (bytes + 255) & ~size_t(255);
        ck_bytes = std::max(ck_bytes, ck_off);
        return measuring ? nullptr : ck_arena + off;
    }
    Act act(int n, int h, int w, int c) {
        Act a;
        a.n = n; a.h = h; a.w = w; a.c = c;
        a.p = alloc(static_cast<size_t>(a.numel()) * es);
        return a;
    }
    float* wptr(int pi) { return w32 + params[pi].off; }
    void* wdev_ptr(int pi) { return static_cast<uint8_t*>(wdev) + params[pi].off * (dt == kF16 ? 2 : 4); }
    void* gptr(int pi) { return static_cast<uint8_t*>(g) + params[pi].off * es; }
    float* bnp(int pi) { return bn32 + params[pi].off; }
    float* bngp(int pi) { return bng + params[pi].off; }

    int add_param(const std::string& name, std::vector<int64_t> shape, int kind, int K = 0, int R = 1, int S = 1,
                  int C = 0) {
        Param p;
        p.name = name;
        p.ref_shape = std::move(shape);
        p.kind = kind;
        if (kind <= 1) {
            p.K = K; p.R = R; p.S = S; p.C = C;
            p.numel = static_cast<int64_t>(K) * R * S * C;
            p.off = n_w;
            n_w += round_up(static_cast<int>(p.numel), 8);  // 16B alignment of every slice
        } else {
            p.numel = p.ref_shape[0];
            p.off = n_bn;
            n_bn += p.numel;
        }
        params.push_back(p);
        return static_cast<int>(params.size()) - 1;
    }

    ConvL conv(const std::string& name, int cin, int cout, int k, int stride, int pad) {
        ConvL c;
        c.p = add_param(name, {cout, cin, k, k}, 0, cout, k, k, cin);
        c.g.K = cout; c.g.R = k; c.g.S = k; c.g.C = cin; c.g.stride = stride; c.g.pad = pad;
        return c;
    }
    NormL norm(const std::string& name, int C, bool relu_or_leaky, bool identity) {
        NormL nl;
        nl.C = C;
        nl.pg = add_param(name + ".gamma", {C}, 2);
        nl.pb = add_param(name + ".beta", {C}, 3);
        nl.mean = static_cast<float*>(alloc(C * 4));
        nl.invstd = static_cast<float*>(alloc(C * 4));
        if (cfg.sync_bn) nl.agg = static_cast<float*>(alloc((2 * C + 1) * 4));
        if (cfg.mode == 0) {
            nl.act = relu_or_leaky ? 1 : 0;
        } else {
            nl.act = 2;
            nl.slope = identity ? 1.0f : cfg.slope;
        }
        return nl;
    }
};

namespace {

struct PScope {
    sdb_det* d;
    int cat;
    cudaEvent_t e0 = nullptr;
    PScope(sdb_det* dd, int c, double flops = 0, double bytes = 0, int nlaunch = 1) : d(dd), cat(c) {
        if (!d->prof.on) return;
        d->prof.flops[c] += flops;
        d->prof.bytes[c] += bytes;
        d->prof.launches[c] += nlaunch;
        e0 = d->prof.get();
        cudaEventRecord(e0, d->ctx->stream);
    }
    ~PScope() {
        if (!e0) return;
        if (nvtx) nvtxRangePop();
        cudaEvent_t e1 = d->prof.get();
        cudaEventRecord(e1, d->ctx->stream);
        d->prof.recs.push_back({cat, {e0, e1}});
        d->prof.labels.push_back(label);
        d->prof.rec_flops.push_back(flops_);
        d->prof.rec_bytes.push_back(bytes_);
    }
    // the record's label; while profiling it also names an NVTX range around
    // the scope's launches (ncu --nvtx --print-nvtx-rename kernel: per-layer
    // counters, tools/ncu_conv_pipe.py)
    void set(std::string l) {
        label = std::move(l);
        if (e0 && !nvtx) {
            nvtxRangePushA(label.c_str());
            nvtx = true;
        }
    }
    std::string label;
    double flops_ = 0, bytes_ = 0;
    bool nvtx = false;
};

std::string shape_label(const char* what, const ConvShape& g) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "%s N%d H%d W%d C%d K%d R%d S%d st%d", what, g.N, g.H, g.W, g.C, g.K, g.R, g.S,
                  g.stride);
    return buf;
}

double conv_flops(const ConvShape& g) {
    return 2.0 * g.N * g.Ho() * g.Wo() * static_cast<double>(g.K) * g.C * g.R * g.S;
}

// ------------------------------------------------------------------ build
void build_stage(sdb_det* d, std::vector<Block>& out, const std::string& pref, int nblocks, int cin, int width,
                 int cout, int stride) {
    for (int b = 0; b < nblocks; ++b) {
        Block bl;
        const std::string p = pref + "." + std::to_string(b);
        const int s = b == 0 ? stride : 1;
        const int ci = b == 0 ? cin : cout;
        bl.c1 = d->conv(p + ".conv1", ci, width, 1, s, 0);
        bl.n1 = d->norm(p + ".bn1", width, true, false);
        bl.c2 = d->conv(p + ".conv2", width, width, 3, 1, 1);
        bl.n2 = d->norm(p + ".bn2", width, true, false);
        bl.c3 = d->conv(p + ".conv3", width, cout, 1, 1, 0);
        bl.n3 = d->norm(p + ".bn3", cout, false, true);
        if (b == 0) {
            bl.has_down = true;
            bl.down = d->conv(p + ".down", ci, cout, 1, s, 0);
            bl.nd = d->norm(p + ".down_bn", cout, false, true);
        }
        out.push_back(bl);
    }
}

// the reference's plan_checkpoints(L) (src/memopt.cpp:76-89): ceil(sqrt(L))
// segments, the first L % segs of them one layer longer; returns the segment
// starts followed by L
std::vector<int> plan_segments(int L) {
    std::vector<int> starts{0};
    const int segs = static_cast<int>(std::ceil(std::sqrt(static_cast<double>(L))));
    const int base = L / segs, rem = L % segs;
    int at = 0;
    for (int j = 0; j + 1 < segs; ++j) {
        at += base + (j < rem ? 1 : 0);
        starts.push_back(at);
    }
    starts.push_back(L);
    return starts;
}

// ck: segment starts (checkpointing) or empty; with segments, every tensor of
// a block goes to the shared arena except the output of a segment's last block
// (the next segment's boundary input, or C4)
void alloc_stage(sdb_det* d, std::vector<Block>& st, Act in, const std::vector<int>& ck = {}) {
    for (size_t i = 0; i < st.size(); ++i) {
        Block& bl = st[i];
        const bool seg = !ck.empty();
        const bool seg_last = seg && std::find(ck.begin(), ck.end(), static_cast<int>(i) + 1) != ck.end();
        if (seg && std::find(ck.begin(), ck.end(), static_cast<int>(i)) != ck.end()) d->ck_off = 0;
        auto mk = [&](int n, int h, int w, int c, bool keep) {
            if (!seg || keep) {
                if (&st == &d->backbone) d->bytes_backbone += static_cast<int64_t>(n) * h * w * c * d->es;
                return d->act(n, h, w, c);
            }
            Act a;
            a.n = n; a.h = h; a.w = w; a.c = c;
            a.p = d->seg_alloc(static_cast<size_t>(a.numel()) * d->es);
            return a;
        };
        bl.in = in;
        auto set = [&](ConvL& c, const Act& x) {
            c.g.N = x.n; c.g.H = x.h; c.g.W = x.w;
        };
        set(bl.c1, in);
        bl.z1 = mk(in.n, bl.c1.g.Ho(), bl.c1.g.Wo(), bl.c1.g.K, false);
        bl.a1 = d->cfg.mode == 0 ? mk(bl.z1.n, bl.z1.h, bl.z1.w, bl.z1.c, false) : bl.z1;
        set(bl.c2, bl.a1);
        bl.z2 = mk(in.n, bl.c2.g.Ho(), bl.c2.g.Wo(), bl.c2.g.K, false);
        bl.a2 = d->cfg.mode == 0 ? mk(bl.z2.n, bl.z2.h, bl.z2.w, bl.z2.c, false) : bl.z2;
        set(bl.c3, bl.a2);
        bl.z3 = mk(in.n, bl.c3.g.Ho(), bl.c3.g.Wo(), bl.c3.g.K, false);
        bl.b3 = d->cfg.mode == 0 ? mk(bl.z3.n, bl.z3.h, bl.z3.w, bl.z3.c, false) : bl.z3;
        if (bl.has_down) {
            set(bl.down, in);
            bl.zd = mk(in.n, bl.down.g.Ho(), bl.down.g.Wo(), bl.down.g.K, false);
            bl.d = d->cfg.mode == 0 ? mk(bl.zd.n, bl.zd.h, bl.zd.w, bl.zd.c, false) : bl.zd;
        }
        bl.out = mk(bl.z3.n, bl.z3.h, bl.z3.w, bl.z3.c, seg_last);
        if (d->cfg.mode != 0 && d->dt == kF16) {
            const size_t nb = static_cast<size_t>(bl.out.numel() / 8);
            if (!seg || seg_last) {
                if (&st == &d->backbone) d->bytes_backbone += static_cast<int64_t>(nb);
                bl.obits = static_cast<uint8_t*>(d->alloc(nb));
            } else {
                bl.obits = static_cast<uint8_t*>(d->seg_alloc(nb));
            }
        }
        d->gbuf_elems = std::max({d->gbuf_elems, in.numel(), bl.z1.numel(), bl.z2.numel(), bl.z3.numel()});
        in = bl.out;
    }
}

void init_params(sdb_det* d) {
    // init_model_params semantics (src/model.cpp:175-195): U(+-sqrt(1/fan_in)),
    // gamma 1, beta 0; seed per tensor = seed*0x9e37 + i*0x85eb (1-based i)
    std::vector<float> wh(static_cast<size_t>(d->n_w), 0.0f), bh(static_cast<size_t>(d->n_bn), 0.0f);
    uint64_t i = 0;
    for (auto& p : d->params) {
        ++i;
        if (p.kind == 2) {
            std::fill(bh.begin() + p.off, bh.begin() + p.off + p.numel, 1.0f);
            continue;
        }
        if (p.kind == 3) continue;
        int64_t fan, n = 1;
        for (int64_t s : p.ref_shape) n *= s;
        if (p.kind == 0) fan = p.ref_shape[1] * p.ref_shape[2] * p.ref_shape[3];
        else fan = p.ref_shape[0];
        const float s = static_cast<float>(std::sqrt(1.0 / static_cast<double>(fan)));
        Rng rng{d->cfg.seed * 0x9e37ull + i * 0x85ebull};
        std::vector<float> ref(static_cast<size_t>(n));
        for (auto& x : ref) x = rng.uniform(-s, s);
        // scatter the reference layout into the device layout
        float* dst = wh.data() + p.off;
        if (p.kind == 0) {
            const int64_t O = p.ref_shape[0], Ci = p.ref_shape[1], kh = p.ref_shape[2], kw = p.ref_shape[3];
            for (int64_t o = 0; o < O; ++o)
                for (int64_t c = 0; c < Ci; ++c)
                    for (int64_t r = 0; r < kh; ++r)
                        for (int64_t q = 0; q < kw; ++q)
                            dst[((o * p.R + r) * p.S + q) * p.C + c] = ref[((o * Ci + c) * kh + r) * kw + q];
        } else {
            const int64_t in = p.ref_shape[0], outc = p.ref_shape[1];
            for (int64_t ii = 0; ii < in; ++ii)
                for (int64_t o = 0; o < outc; ++o) dst[o * p.C + ii] = ref[ii * outc + o];
        }
    }
    // stream-ordered copies: a pageable cudaMemcpy may return before its DMA
    // lands, and the cast below runs on the (non-blocking) context stream
    cudaStream_t st0 = d->ctx->stream;
    CK(cudaMemcpyAsync(d->w32, wh.data(), wh.size() * 4, cudaMemcpyHostToDevice, st0));
    CK(cudaMemcpyAsync(d->bn32, bh.data(), bh.size() * 4, cudaMemcpyHostToDevice, st0));
    CK(cudaMemsetAsync(d->v32, 0, wh.size() * 4, st0));
    CK(cudaMemsetAsync(d->bnv, 0, bh.size() * 4, st0));
    if (d->dt == kF16) CK(cast_f32_f16(d->w32, static_cast<__half*>(d->wdev), d->n_w, d->ctx->stream));
    CK(cudaStreamSynchronize(d->ctx->stream));
}

size_t max_ws(sdb_det* d) {
    size_t m = 1 << 20;
    auto conv_ws = [&](const ConvL& c) { m = std::max(m, conv_wgrad_workspace(c.g, d->dt)); };
    auto norm_ws = [&](const NormL& n, int64_t rows) { m = std::max(m, norm_workspace_bytes(rows, n.C)); };
    conv_ws(d->stem);
    if (d->stem_gemm) conv_ws(d->stem2);
    norm_ws(d->stem_n, static_cast<int64_t>(d->stem_z.n) * d->stem_z.h * d->stem_z.w);
    for (auto* st : {&d->backbone, &d->head})
        for (auto& b : *st) {
            conv_ws(b.c1); conv_ws(b.c2); conv_ws(b.c3);
            norm_ws(b.n1, static_cast<int64_t>(b.z1.n) * b.z1.h * b.z1.w);
            norm_ws(b.n2, static_cast<int64_t>(b.z2.n) * b.z2.h * b.z2.w);
            norm_ws(b.n3, static_cast<int64_t>(b.z3.n) * b.z3.h * b.z3.w);
            if (b.has_down) conv_ws(b.down);
        }
    conv_ws(d->rpn_conv); conv_ws(d->rpn_cls); conv_ws(d->rpn_bbox); conv_ws(d->fc_cls); conv_ws(d->fc_bbox);
    m = std::max(m, proposal_workspace_bytes(d->cfg.batch, d->nA, d->cfg.pre_nms));
    m = std::max(m, anchor_target_workspace_bytes(d->cfg.batch, d->nA, d->cfg.max_gt));
    m = std::max(m, roialign_bwd_workspace(d->R, d->fh, d->fw, d->P, d->roi_step, d->cfg.batch));
    return m;
}

// ------------------------------------------------------------------ forward helpers
void conv_fwd(sdb_det* d, const ConvL& c, const Act& x, const Act& y, bool want_stats = false) {
    PScope ps(d, P_FPROP, conv_flops(c.g));
    if (d->prof.on) { ps.set(shape_label("fprop", c.g)); ps.flops_ = conv_flops(c.g); }
    CK(conv_fprop(c.g, d->dt, x.p, d->wdev_ptr(c.p), y.p, d->ctx->stream,
                  want_stats && d->cst.buf ? &d->cst : nullptr));
    if (!(want_stats && d->cst.buf)) d->cst.produced = 0;
}

void norm_fwd(sdb_det* d, const NormL& n, const Act& z, const Act& a) {
    const int64_t rows = static_cast<int64_t>(z.n) * z.h * z.w;
    if (d->cst.produced) {
        // statistics came out of the producing fprop's epilogue: finalize + apply
        PScope ps(d, P_NORM_F, 0, 2.0 * d->es * z.numel(), 2);
        if (d->prof.on && std::getenv("SDB_PROFILE_VERBOSE")) {
            ps.set("norm_fwd(fused stats) rows " + std::to_string(rows) + " C " + std::to_string(n.C));
            ps.bytes_ = 2.0 * d->es * z.numel();
        }
        CK(bn_forward_conv_stats(d->dt, z.p, d->bnp(n.pg), d->bnp(n.pb), a.p, n.mean, n.invstd, rows, n.C, d->cfg.eps,
                                 n.act, n.slope, d->cst, d->ctx->stream));
        d->cst.produced = 0;
        return;
    }
    PScope ps(d, P_NORM_F, 0, 2.0 * d->es * z.numel(), 3);
    if (d->prof.on && std::getenv("SDB_PROFILE_VERBOSE")) {
        ps.set("norm_fwd rows " + std::to_string(rows) + " C " + std::to_string(n.C));
        ps.bytes_ = 3.0 * d->es * z.numel();
    }
    if (n.agg) {
        // SyncBN (src/syncbn.cpp:21-70): this rank's float sums, summed over the
        // ranks on the step stream, then statistics + apply from the global sums
        CK(syncbn_local_sums(d->dt, z.p, rows, n.C, n.agg, d->ws, d->ctx->stream));
        if (d->comm_on) CKC(comm_allreduce(d->ctx, n.agg, 2 * n.C + 1, kF32, 0, d->ctx->stream));
        CK(syncbn_forward_finish(d->dt, z.p, d->bnp(n.pg), d->bnp(n.pb), a.p, n.mean, n.invstd, n.agg, rows, n.C,
                                 d->cfg.eps, n.act, d->ctx->stream));
        return;
    }
    CK(bn_forward(d->dt, z.p, d->bnp(n.pg), d->bnp(n.pb), a.p, n.mean, n.invstd, rows, n.C, d->cfg.eps, n.act,
                  n.slope, d->ws, d->ctx->stream));
}

// dz from da for a norm layer; y = a (stored output), x = z (pre-norm, mode 0 only)
void norm_bwd(sdb_det* d, const NormL& n, const Act& z, const Act& a, const void* da, void* dz) {
    const int64_t rows = static_cast<int64_t>(z.n) * z.h * z.w;
    PScope ps(d, P_NORM_B, 0, 3.0 * d->es * z.numel(), 3);
    if (d->prof.on && std::getenv("SDB_PROFILE_VERBOSE")) {
        ps.set("norm_bwd rows " + std::to_string(rows) + " C " + std::to_string(n.C));
        ps.bytes_ = 5.0 * d->es * z.numel();
    }
    if (n.agg) {
        // SyncBN backward (src/syncbn.cpp:72-117): [sum dy, sum dy*xhat] summed over
        // the ranks, coefficients with the forward's global count
        const void* mask = n.act == 1 ? a.p : nullptr;
        CK(syncbn_backward_local_sums(d->dt, da, z.p, mask, n.mean, n.invstd, d->sbn_red, rows, n.C, d->ws,
                                      d->ctx->stream));
        if (d->comm_on) CKC(comm_allreduce(d->ctx, d->sbn_red, 2 * n.C, kF32, 0, d->ctx->stream));
        CK(syncbn_backward_finish(d->dt, da, z.p, mask, d->bnp(n.pg), n.mean, n.invstd, d->sbn_red, n.agg, dz,
                                  d->bngp(n.pg), d->bngp(n.pb), rows, n.C, d->ws, d->ctx->stream));
    } else if (d->cfg.mode == 0) {
        CK(bn_backward(d->dt, da, z.p, n.act == 1 ? a.p : nullptr, d->bnp(n.pg), n.mean, n.invstd, dz,
                       d->bngp(n.pg), d->bngp(n.pb), rows, n.C, d->ws, d->ctx->stream));
    } else if (d->cst_b.produced && d->cst_b.bs_y == a.p) {
        // statistics came out of the dgrad epilogue that produced da: finalize + apply
        CK(iabn_backward_conv_stats(d->dt, da, a.p, d->bnp(n.pg), d->bnp(n.pb), n.invstd, dz, d->bngp(n.pg),
                                    d->bngp(n.pb), rows, n.C, n.slope, d->cst_b, static_cast<float*>(d->ws),
                                    d->ctx->stream));
        d->cst_b.produced = 0;
    } else {
        CK(iabn_backward(d->dt, da, a.p, d->bnp(n.pg), d->bnp(n.pb), n.mean, n.invstd, dz, d->bngp(n.pg),
                         d->bngp(n.pb), rows, n.C, n.slope, d->ws, d->ctx->stream));
    }
}

// the shortcut branch of a downsampling block on d->bst: fused-statistics fprop
// + InPlace-ABN (in place), its own ConvStats; joined before the residual add
void shortcut_fwd_branch(sdb_det* d, Block& b) {
    CK(cudaEventRecord(d->ev_b_fork, d->ctx->stream));
    CK(cudaStreamWaitEvent(d->bst, d->ev_b_fork, 0));
    CK(conv_fprop(b.down.g, d->dt, b.in.p, d->wdev_ptr(b.down.p), b.zd.p, d->bst, &d->cst2));
    const int64_t rows = static_cast<int64_t>(b.zd.n) * b.zd.h * b.zd.w;
    if (d->cst2.produced)
        CK(bn_forward_conv_stats(d->dt, b.zd.p, d->bnp(b.nd.pg), d->bnp(b.nd.pb), b.d.p, b.nd.mean, b.nd.invstd, rows,
                                 b.nd.C, d->cfg.eps, b.nd.act, b.nd.slope, d->cst2, d->bst));
    else
        CK(bn_forward(d->dt, b.zd.p, d->bnp(b.nd.pg), d->bnp(b.nd.pb), b.d.p, b.nd.mean, b.nd.invstd, rows, b.nd.C,
                      d->cfg.eps, b.nd.act, b.nd.slope, d->ws2, d->bst));
    d->cst2.produced = 0;
    CK(cudaEventRecord(d->ev_b_join, d->bst));
}

void block_fwd(sdb_det* d, Block& b) {
    // concurrent shortcut branch: fp16 InPlace-ABN graph steps (not the eager profile)
    const bool branch = b.has_down && d->bst && !d->prof.on && b.n3.act == 2;
    if (branch) shortcut_fwd_branch(d, b);
    conv_fwd(d, b.c1, b.in, b.z1, true);
    norm_fwd(d, b.n1, b.z1, b.a1);
    conv_fwd(d, b.c2, b.a1, b.z2, true);
    norm_fwd(d, b.n2, b.z2, b.a2);
    conv_fwd(d, b.c3, b.a2, b.z3, true);
    if (b.n3.act == 2) {
        // InPlace-ABN bn3: statistics now, the apply fused with the residual
        // add + leaky that closes the block (one pass: reads z3 + shortcut,
        // writes y3 in place and the block output)
        const int64_t rows = static_cast<int64_t>(b.z3.n) * b.z3.h * b.z3.w;
        {
            PScope ps(d, P_NORM_F, 0, 1.0 * d->es * b.z3.numel(), 2);
            if (d->prof.on && std::getenv("SDB_PROFILE_VERBOSE")) {
                ps.set(std::string(d->cst.produced ? "norm_stats3(fused) rows " : "norm_stats3 rows ") +
                       std::to_string(rows) + " C " + std::to_string(b.n3.C));
                ps.bytes_ = 1.0 * d->es * b.z3.numel();
            }
            if (d->cst.produced) {
                CK(bn_forward_conv_stats(d->dt, b.z3.p, nullptr, nullptr, nullptr, b.n3.mean, b.n3.invstd, rows,
                                         b.n3.C, d->cfg.eps, b.n3.act, 1.0f, d->cst, d->ctx->stream));
                d->cst.produced = 0;
            } else {
                CK(bn_forward_stats(d->dt, b.z3.p, b.n3.mean, b.n3.invstd, rows, b.n3.C, d->cfg.eps, b.n3.act, d->ws,
                                    d->ctx->stream));
            }
        }
        const Act* sc = &b.in;
        if (b.has_down) {
            if (branch) {
                CK(cudaStreamWaitEvent(d->ctx->stream, d->ev_b_join, 0));
            } else {
                conv_fwd(d, b.down, b.in, b.zd, true);
                norm_fwd(d, b.nd, b.zd, b.d);
            }
            sc = &b.d;
        }
        PScope ps(d, P_NORM_F, 0, 4.0 * d->es * b.out.numel());
        if (d->prof.on && std::getenv("SDB_PROFILE_VERBOSE")) {
            ps.set("norm_apply_add rows " + std::to_string(rows) + " C " + std::to_string(b.n3.C));
            ps.bytes_ = 4.0 * d->es * b.out.numel();
        }
        if (d->head_pool_fuse && &b == &d->head.back()) {
            CK(bn_apply_add_act_pool(d->dt, b.z3.p, d->bnp(b.n3.pg), d->bnp(b.n3.pb), b.n3.mean, b.n3.invstd, b.b3.p,
                                     sc->p, d->pooled.p, b.out.h * b.out.w, rows, b.n3.C, b.n3.slope, 2,
                                     d->cfg.slope, d->ctx->stream, b.obits));
            return;
        }
        CK(bn_apply_add_act(d->dt, b.z3.p, d->bnp(b.n3.pg), d->bnp(b.n3.pb), b.n3.mean, b.n3.invstd, b.b3.p, sc->p,
                            b.out.p, rows, b.n3.C, b.n3.slope, 2, d->cfg.slope, d->ctx->stream, b.obits));
        return;
    }
    norm_fwd(d, b.n3, b.z3, b.b3);
    const Act* sc = &b.in;
    if (b.has_down) {
        conv_fwd(d, b.down, b.in, b.zd, true);
        norm_fwd(d, b.nd, b.zd, b.d);
        sc = &b.d;
    }
    PScope ps(d, P_ELEM, 0, 3.0 * d->es * b.out.numel());
    CK(add_act(d->dt, b.b3.p, sc->p, b.out.p, b.out.numel(), d->cfg.mode == 0 ? 1 : 2, d->cfg.slope, d->ctx->stream));
}

// ------------------------------------------------------------------ backward helpers
void dgrad(sdb_det* d, const ConvL& c, const void* dy, void* dx, int accumulate, const void* addend = nullptr,
           const void* mask = nullptr, float mask_neg = 0.0f, const uint8_t* mask_bits = nullptr,
           ConvStats* bstats = nullptr) {
    PScope ps(d, P_DGRAD, conv_flops(c.g), 0, c.g.stride * c.g.stride);
    if (d->prof.on) {
        ps.set(shape_label(mask_bits ? "dgrad+res" : (bstats ? "dgrad+bstats" : "dgrad"), c.g));
        ps.flops_ = conv_flops(c.g);
    }
    CK(conv_dgrad(c.g, d->dt, dy, d->wdev_ptr(c.p), dx, accumulate, d->ctx->stream, addend, mask, mask_neg,
                  mask_bits, bstats));
}

// the dgrad that writes the output gradient of InPlace-ABN layer n (stored
// output y): reduce n's backward statistics in its epilogue (fp16 IABN mode)
ConvStats* bstats_for(sdb_det* d, const NormL& n, const Act& y) {
    if (!d->cst_b.buf || d->cfg.mode != 1 || std::getenv("SDB_NO_FUSED_BWD_STATS")) return nullptr;
    d->cst_b.bs_y = y.p;
    d->cst_b.bs_gamma = d->bnp(n.pg);
    d->cst_b.bs_beta = d->bnp(n.pb);
    d->cst_b.bs_slope = n.slope;
    return &d->cst_b;
}

struct Bwd {
    sdb_det* d;
    int64_t issued_lo;  // lowest g offset whose bucket has been issued
    size_t next_bucket = 0;
    bool side = false;  // wgrads on d->wst (not while profiling: per-category events live on the main stream)
    int slot = -1;      // dz ring slot handed out by dz_buf and not yet consumed by a wgrad
};

// where the next norm backward writes the dz that a wgrad will read: a ring slot
// (waiting for the wgrad that last read it) when wgrads run on the side stream
void* dz_buf(Bwd& B, void* fallback) {
    sdb_det* d = B.d;
    if (!B.side) return fallback;
    const int k = d->dzr_next;
    d->dzr_next = (k + 1) % d->dzr_n;
    if (d->dzr_busy[k]) CK(cudaStreamWaitEvent(d->ctx->stream, d->dzr_ev[k], 0));
    d->dzr_busy[k] = false;
    B.slot = k;
    return d->dzr[k];
}

// allreduce of gradient bucket b on the comm stream once `st` reaches this
// point.  fp16 buckets are AVERAGED (ncclAvg: NCCL pre-multiplies each rank's
// values by 1/K, then sums), so the reduced value stays in range whenever
// every rank's is -- overflow detection does not depend on K -- and the
// optimizer divides by the loss scale only; fp32 buckets are summed and the
// optimizer divides by scale*K (src/trainer.cpp:86-94).
void issue_bucket_allreduce(sdb_det* d, size_t b, cudaStream_t st) {
    const auto [lo, hi] = d->buckets[b];
    cudaEvent_t ev = d->bucket_ev[b];
    CK(cudaEventRecord(ev, st));
    CK(cudaStreamWaitEvent(d->comm, ev, 0));
    if (d->shard)
        CKC(comm_reduce_scatter(d->ctx, static_cast<uint8_t*>(d->g) + lo * d->es, (hi - lo) / d->ctx->world, d->dt, 1,
                                d->comm));
    else
        CKC(comm_allreduce(d->ctx, static_cast<uint8_t*>(d->g) + lo * d->es, hi - lo, d->dt, d->dt == kF16, d->comm));
}

// non-deferred wgrads (fp32 modes): buckets are issued in plan order as the
// backward pass walks past their lower edge
void grads_ready(Bwd& B, int pi) {
    sdb_det* d = B.d;
    if (!d->comm_on) return;
    const int64_t off = d->params[pi].off;
    while (B.next_bucket < d->buckets.size() && off <= d->buckets[B.next_bucket].first) {
        PScope ps(d, P_COMM, 0, static_cast<double>(d->buckets[B.next_bucket].second - d->buckets[B.next_bucket].first) * d->es);
        issue_bucket_allreduce(d, B.next_bucket, d->ctx->stream);
        ++B.next_bucket;
    }
}

// deferred wgrads: bucket b is complete once the wgrad of each of its
// parameters has been issued; its split-K partials are then reduced by one
// batched launch on the stream that ran those wgrads (stream order covers
// them), the stem's GEMM-form gradient is folded back, and the bucket goes to
// the comm stream.  The job tables are static (fixed shapes and buffers):
// uploaded once, from the first (eager) step.
void flush_bucket(sdb_det* d, int b, cudaStream_t st) {
    auto& T = d->btab[b];
    auto& J = d->bjobs[b];
    if (!T.jobs) {
        std::vector<int> start(J.size());
        int tot = 0;
        for (size_t k = 0; k < J.size(); ++k) {
            start[k] = tot;
            tot += wgrad_job_tiles(J[k]);
        }
        T.jobs = static_cast<WgradJob*>(d->alloc(J.size() * sizeof(WgradJob)));
        T.tiles = static_cast<int*>(d->alloc(start.size() * sizeof(int)));
        CK(cudaMemcpyAsync(T.jobs, J.data(), J.size() * sizeof(WgradJob), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(T.tiles, start.data(), start.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
        T.njobs = static_cast<int>(J.size());
        T.total = tot;
    } else if (static_cast<int>(J.size()) != T.njobs) {
        throw std::runtime_error("wgrad job table changed between steps");
    }
    J.clear();
    {
        PScope ps(d, P_WGRAD, 0, 0, 1);
        CK(wgrad_reduce_batched(T.jobs, T.tiles, T.njobs, T.total, st, d->flag));
        if (d->stem_gemm && d->bucket_of[d->stem.p] == b)
            CK(stem_weights(d->stem_dw2, 64, 8, d->gptr(d->stem.p), 1, st));
    }
    if (d->comm_on) {
        PScope ps(d, P_COMM, 0, static_cast<double>(d->buckets[b].second - d->buckets[b].first) * d->es);
        issue_bucket_allreduce(d, static_cast<size_t>(b), st);
    }
}

void job_issued(sdb_det* d, int pi, const WgradJob& job, cudaStream_t st) {
    const int b = d->bucket_of.at(pi);
    if (b < 0) throw std::runtime_error("wgrad of a parameter outside the bucket plan");
    d->bjobs[b].push_back(job);
    if (--d->bucket_left[b] == 0) flush_bucket(d, b, st);
}

void conv_wgrad_to(Bwd& B, const ConvL& c, const Act& x, const void* dy, void* dw_override = nullptr,
                   bool ready = true) {
    sdb_det* d = B.d;
    void* dwp = dw_override ? dw_override : d->gptr(c.p);
    {
    PScope ps(d, P_WGRAD, conv_flops(c.g), 0, 2);
    if (d->prof.on) { ps.set(shape_label("wgrad", c.g)); ps.flops_ = conv_flops(c.g); }
    if (d->defer_wgrad) {
        auto it = d->wg_off.find(c.p);
        if (it == d->wg_off.end()) throw std::runtime_error("wgrad arena: unknown conv");
        cudaStream_t ws = d->ctx->stream;
        if (B.side) {
            CK(cudaEventRecord(d->wev_fork, ws));
            CK(cudaStreamWaitEvent(d->wst, d->wev_fork, 0));
            ws = d->wst;
        }
        WgradJob job{};
        CK(conv_wgrad_deferred(c.g, d->dt, x.p, dy, dwp, d->wg_arena + it->second,
                               conv_wgrad_workspace(c.g, d->dt), ws, &job));
        if (B.side && B.slot >= 0 && dy == d->dzr[B.slot]) {
            CK(cudaEventRecord(d->dzr_ev[B.slot], d->wst));
            d->dzr_busy[B.slot] = true;
            B.slot = -1;
        }
        job_issued(d, c.p, job, ws);
        return;
    }
    CK(conv_wgrad(c.g, d->dt, x.p, dy, dwp, d->ws, d->ws_bytes, d->ctx->stream));
    }
    if (ready) grads_ready(B, c.p);
}

// the stem's GEMM-form wgrad into dW' (stem_dw2); without the deferred reduce
// it is folded into the gradient right away, else by its bucket's flush
void stem_wgrad_to(Bwd& B, const ConvL& c2, void* x2, const void* dy) {
    sdb_det* d = B.d;
    Act xa{};
    xa.p = x2;
    conv_wgrad_to(B, c2, xa, dy, d->stem_dw2, false);
    if (!d->defer_wgrad) {
        CK(stem_weights(d->stem_dw2, 64, 8, d->gptr(d->stem.p), 1, d->ctx->stream));
        grads_ready(B, d->stem.p);
    }
}

// backward of a bottleneck.  dS = gradient at the residual add node (the
// block's output activation already back-propagated: the producer of dS applied
// the activation mask in its dgrad epilogue).  Writes the gradient wrt b.in into
// dx; when b.in is itself a residual-block output (in_mask != null) the final
// dgrad epilogue applies that block's activation mask too, so dx is the next
// block's dS.  Uses scratch buffers s1, s2.
void block_bwd(Bwd& B, Block& b, const void* dS, void* dx, void* s1, void* s2, const void* in_mask,
               const uint8_t* in_bits) {
    sdb_det* d = B.d;
    const float neg = d->cfg.mode == 0 ? 0.0f : d->cfg.slope;
    // shortcut first (its params come last in the block's pack order)
    void* z;
    const bool branch = b.has_down && d->bst && d->dzb && B.side && d->cfg.mode == 1;
    if (branch) {
        // on d->bst, next to the conv3..conv1 chain: the shortcut's IABN backward
        // (statistics pass), its wgrad (side stream) and its dgrad into dx; the
        // chain's final dgrad accumulates onto dx after the join
        cudaStream_t bs = d->bst;
        CK(cudaEventRecord(d->ev_b_fork, d->ctx->stream));
        CK(cudaStreamWaitEvent(bs, d->ev_b_fork, 0));
        if (d->dzb_busy) CK(cudaStreamWaitEvent(bs, d->ev_dzb, 0));
        const int64_t rows = static_cast<int64_t>(b.zd.n) * b.zd.h * b.zd.w;
        CK(iabn_backward(d->dt, dS, b.d.p, d->bnp(b.nd.pg), d->bnp(b.nd.pb), b.nd.mean, b.nd.invstd, d->dzb,
                         d->bngp(b.nd.pg), d->bngp(b.nd.pb), rows, b.nd.C, b.nd.slope, d->ws2, bs));
        CK(cudaEventRecord(d->ev_b2_fork, bs));
        CK(cudaStreamWaitEvent(d->wst, d->ev_b2_fork, 0));
        WgradJob job{};
        CK(conv_wgrad_deferred(b.down.g, d->dt, b.in.p, d->dzb, d->gptr(b.down.p), d->wg_arena + d->wg_off.at(b.down.p),
                               conv_wgrad_workspace(b.down.g, d->dt), d->wst, &job));
        CK(cudaEventRecord(d->ev_dzb, d->wst));
        d->dzb_busy = true;
        job_issued(d, b.down.p, job, d->wst);
        CK(conv_dgrad(b.down.g, d->dt, d->dzb, d->wdev_ptr(b.down.p), dx, 0, bs));
        CK(cudaEventRecord(d->ev_b_join, bs));
    } else if (b.has_down) {
        z = dz_buf(B, s1);
        norm_bwd(d, b.nd, b.zd, b.d, dS, z);
        conv_wgrad_to(B, b.down, b.in, z);
        dgrad(d, b.down, z, dx, 0);
    }
    z = dz_buf(B, s1);
    if (d->head_pool_bwd && &b == &d->head.back()) {
        // dS is the masked average-pool gradient: formed inside bn3's statistics
        // pass from the pooled gradient and the sign bitmap (and stored there
        // for the residual fan-in below), again inside the apply pass
        const int64_t rows = static_cast<int64_t>(b.z3.n) * b.z3.h * b.z3.w;
        PScope ps(d, P_NORM_B, 0, d->es * (4.0 * b.z3.numel()) + b.z3.numel() / 4.0, 3);
        CK(iabn_backward_pooled(d->dt, d->dpool_cur, b.obits, b.z3.h * b.z3.w, neg, b.b3.p, d->bnp(b.n3.pg),
                                d->bnp(b.n3.pb), b.n3.invstd, const_cast<void*>(dS), z, d->bngp(b.n3.pg),
                                d->bngp(b.n3.pb), rows, b.n3.C, b.n3.slope, d->ws, d->ctx->stream));
    } else {
        norm_bwd(d, b.n3, b.z3, b.b3, dS, z);
    }
    conv_wgrad_to(B, b.c3, b.a2, z);
    dgrad(d, b.c3, z, s2, 0, nullptr, nullptr, 0.0f, nullptr, bstats_for(d, b.n2, b.a2));
    z = dz_buf(B, s1);
    norm_bwd(d, b.n2, b.z2, b.a2, s2, z);
    conv_wgrad_to(B, b.c2, b.a1, z);
    dgrad(d, b.c2, z, s2, 0, nullptr, nullptr, 0.0f, nullptr, bstats_for(d, b.n1, b.a1));
    z = dz_buf(B, s1);
    norm_bwd(d, b.n1, b.z1, b.a1, s2, z);
    conv_wgrad_to(B, b.c1, b.in, z);
    // residual fan-in in the dgrad epilogue: dx = conv1^T(dz1) + (down-path dx | identity dS),
    // then the previous block's activation mask
    if (branch) CK(cudaStreamWaitEvent(d->ctx->stream, d->ev_b_join, 0));
    if (b.has_down) dgrad(d, b.c1, z, dx, 1, nullptr, in_mask, neg, in_bits);
    else dgrad(d, b.c1, z, dx, 1, dS, in_mask, neg, in_bits);
}

// RPN losses + RPN head backward on the side stream (see sdb_det::ev_rpn_fork);
// leaves the RPN-conv input gradient in d->drpn_side
void rpn_branch_side(sdb_det* d) {
    const auto& cf = d->cfg;
    cudaStream_t s2 = d->wst;
    LossArgs la{d->scale, d->losses, 0};
    CK(sigmoid_bce(d->dt, d->rpn_logits.p, static_cast<int64_t>(d->n_loc) * cf.batch, d->A, d->A_pad, d->a_labels,
                   d->d_rpn_logits, la, d->ws_at, s2));
    la.slot = 1;
    CK(rpn_smooth_l1(d->dt, d->rpn_deltas.p, static_cast<int64_t>(d->n_loc) * cf.batch, d->A, d->A_pad, d->a_labels,
                     d->a_targets, 1.0 / 9.0, static_cast<double>(cf.rpn_batch) * cf.batch, d->d_rpn_deltas, la,
                     d->ws_at, s2));
    auto wgrad = [&](const ConvL& c, const void* x, const void* dy) {
        WgradJob job{};
        CK(conv_wgrad_deferred(c.g, d->dt, x, dy, d->gptr(c.p), d->wg_arena + d->wg_off.at(c.p),
                               conv_wgrad_workspace(c.g, d->dt), s2, &job));
        job_issued(d, c.p, job, s2);
    };
    wgrad(d->rpn_bbox, d->rpn_a.p, d->d_rpn_deltas);
    wgrad(d->rpn_cls, d->rpn_a.p, d->d_rpn_logits);
    // the RPN ReLU backward folded into the dgrad that writes drpn last (K % 64 == 0)
    const bool bbox_last = (d->rpn_bbox.g.K % 64) == 0;
    const ConvL& r_first = bbox_last ? d->rpn_cls : d->rpn_bbox;
    const ConvL& r_last = bbox_last ? d->rpn_bbox : d->rpn_cls;
    CK(conv_dgrad(r_first.g, d->dt, bbox_last ? d->d_rpn_logits : d->d_rpn_deltas, d->wdev_ptr(r_first.p),
                  d->drpn_side, 0, s2));
    if ((r_last.g.K % 64) == 0) {
        CK(conv_dgrad(r_last.g, d->dt, bbox_last ? d->d_rpn_deltas : d->d_rpn_logits, d->wdev_ptr(r_last.p),
                      d->drpn_side, 1, s2, nullptr, d->rpn_a.p, 0.0f));
    } else {
        CK(conv_dgrad(r_last.g, d->dt, bbox_last ? d->d_rpn_deltas : d->d_rpn_logits, d->wdev_ptr(r_last.p),
                      d->drpn_side, 1, s2));
        CK(act_bwd(d->dt, d->drpn_side, d->rpn_a.p, d->drpn_side, d->rpn_a.numel(), 0.0f, s2));
    }
    wgrad(d->rpn_conv, d->c4.p, d->drpn_side);
}

// ------------------------------------------------------------------ the step
void run_step(sdb_det* d) {
    cudaStream_t st = d->ctx->stream;
    const auto& cf = d->cfg;
    const bool side = d->side_wgrad && !d->prof.on;
    d->bucket_left = d->bucket_nparams;
    for (auto& j : d->bjobs) j.clear();
    // the overflow flag is OR-ed by the bucket reduces (deferred fp16 wgrads)
    // and the BN-gradient check; zeroed before any of them can run
    CK(cudaMemsetAsync(d->flag, 0, sizeof(int), st));
    AnchorTargetArgs at{};
    at.anchors = d->anchors; at.nA = d->nA; at.n_img = cf.batch; at.gt = d->gt; at.gt_stride = cf.max_gt;
    at.gt_count = d->gt_count; at.img_h = static_cast<float>(cf.img_h); at.img_w = static_cast<float>(cf.img_w);
    at.keys = d->keys; at.fg_thr = cf.rpn_fg_thr; at.bg_thr = cf.rpn_bg_thr; at.batch = cf.rpn_batch;
    at.fg_cap = static_cast<int>(cf.rpn_fg_frac * cf.rpn_batch); at.labels = d->a_labels; at.targets = d->a_targets;
    if (side) {
        CK(cudaEventRecord(d->ev_at_fork, st));
        CK(cudaStreamWaitEvent(d->wst, d->ev_at_fork, 0));
        CK(anchor_targets(at, d->ws_at, d->wst));
        CK(cudaEventRecord(d->ev_at_join, d->wst));
    }
    // ---- forward: backbone
    if (d->stem_gemm) {
        {
            PScope ps(d, P_ELEM, 0, 2.0 * (d->img.numel() + static_cast<double>(d->stem2.g.W) * 192), 3);
            if (d->prof.on) ps.set("stem im2col + weight pack");
            CK(stem_weights(d->wdev_ptr(d->stem.p), 64, 8, d->stem_w2, 0, st));
            CK(stem_im2col(d->img.p, d->img.n, d->img.h, d->img.w, 8, d->stem_z.h, d->stem_z.w, 2, 3, d->stem_x2,
                           st));
        }
        PScope ps(d, P_FPROP, conv_flops(d->stem2.g));
        if (d->prof.on) { ps.set(shape_label("fprop(stem gemm)", d->stem2.g)); ps.flops_ = conv_flops(d->stem2.g); }
        CK(conv_fprop(d->stem2.g, d->dt, d->stem_x2, d->stem_w2, d->stem_z.p, st, d->cst.buf ? &d->cst : nullptr));
    } else {
        conv_fwd(d, d->stem, d->img, d->stem_z, true);
    }
    norm_fwd(d, d->stem_n, d->stem_z, d->stem_a);
    { PScope ps(d, P_POOL, 0, d->es * (d->stem_a.numel() + d->pool.numel()));
    CK(maxpool_fwd(d->dt, d->stem_a.p, d->stem_a.n, d->stem_a.h, d->stem_a.w, d->stem_a.c, 3, 2, 1, d->pool.p,
                   d->pool_arg, st)); }
    for (auto& b : d->backbone) block_fwd(d, b);
    // ---- RPN head
    conv_fwd(d, d->rpn_conv, d->c4, d->rpn_z);
    { PScope ps(d, P_ELEM, 0, 2.0 * d->es * d->rpn_z.numel());
    CK(relu_fwd(d->dt, d->rpn_z.p, d->rpn_a.p, d->rpn_a.numel(), st)); }
    conv_fwd(d, d->rpn_cls, d->rpn_a, d->rpn_logits);
    conv_fwd(d, d->rpn_bbox, d->rpn_a, d->rpn_deltas);
    if (side) {
        // wst already holds the anchor targets; add the RPN losses and head backward
        CK(cudaEventRecord(d->ev_rpn_fork, st));
        CK(cudaStreamWaitEvent(d->wst, d->ev_rpn_fork, 0));
        rpn_branch_side(d);
        CK(cudaEventRecord(d->ev_rpn_join, d->wst));
    }
    // ---- targets and proposals (no gradient)
    if (!side) { PScope ps(d, P_TARGETS, 0, 0, 5); CK(anchor_targets(at, d->ws, st)); }
    ProposalArgs pa{};
    pa.logits = d->rpn_logits.p; pa.deltas = d->rpn_deltas.p; pa.dtype = d->dt; pa.anchors = d->anchors;
    pa.n_img = cf.batch; pa.n_loc = d->n_loc; pa.A = d->A; pa.A_pad = d->A_pad; pa.pre_k = cf.pre_nms;
    pa.post_k = cf.post_nms; pa.iou_thr = cf.nms_iou; pa.img_h = static_cast<float>(cf.img_h);
    pa.img_w = static_cast<float>(cf.img_w); pa.clip_dw = static_cast<float>(std::log(1000.0 / 16.0));
    pa.rois = d->props; pa.roi_scores = nullptr; pa.keep_pos = d->keep_pos; pa.count = d->prop_count;
    {
        // algorithmic bytes: objectness + deltas read, anchors read, the pre-NMS
        // candidate boxes written and read once, the kept boxes written
        const double kk = std::min<double>(cf.pre_nms, static_cast<double>(d->nA));
        const double by = static_cast<double>(cf.batch) * d->n_loc * d->A_pad * 5.0 * d->es + 16.0 * d->nA +
                          cf.batch * (32.0 * kk + 16.0 * cf.post_nms);
        PScope ps(d, P_PROPOSAL, 0, by, 3);
        CK(rpn_proposals(pa, d->ws, st));
    }
    ProposalTargetArgs pt{};
    pt.proposals = d->props; pt.prop_stride = cf.post_nms; pt.prop_count = d->prop_count; pt.gt = d->gt;
    pt.gt_cls = d->gt_cls; pt.gt_stride = cf.max_gt; pt.gt_count = d->gt_count; pt.keys = d->keys + cf.batch;
    pt.fg_thr = cf.roi_fg_thr; pt.bg_hi = cf.roi_bg_hi; pt.bg_lo = cf.roi_bg_lo; pt.batch = cf.roi_batch;
    pt.fg_cap = static_cast<int>(std::llround(cf.roi_fg_frac * cf.roi_batch)); pt.n_img = cf.batch;
    pt.work_flag = d->pt_flag; pt.work_arg = d->pt_arg; pt.work_stride = cf.post_nms + cf.max_gt;
    pt.out_rois = d->rois; pt.out_labels = d->roi_labels; pt.out_targets = d->roi_targets; pt.out_src = nullptr;
    pt.out_count = d->roi_count;
    { PScope ps(d, P_TARGETS, 0, 0, 1); CK(proposal_targets(pt, st)); }
    // ---- RoI head
    const float sscale = 1.0f / 16.0f;
    { PScope ps(d, P_ROI_F, 0, static_cast<double>(d->es) * (d->roi_feat.numel() + d->c4.numel()));
    CK(roialign_fwd(d->dt, d->c4.p, d->c4.n, d->c4.h, d->c4.w, d->c4.c, d->rois, d->R, d->P, sscale,
                    cf.sampling_ratio, d->roi_feat.p, st, d->roi_step)); }
    for (auto& b : d->head) block_fwd(d, b);
    if (!d->head_pool_fuse) {
        PScope ps(d, P_POOL, 0, static_cast<double>(d->es) * d->head_out.numel());
        CK(avgpool_fwd(d->dt, d->head_out.p, d->R, d->head_out.h * d->head_out.w, d->feat_c, d->pooled.p, st));
    }
    conv_fwd(d, d->fc_cls, d->pooled, d->cls_logits);
    conv_fwd(d, d->fc_bbox, d->pooled, d->bbox_pred);
    // ---- losses (scale folded into backward)
    CK(cudaMemcpyAsync(d->scale_used, d->scale, 8, cudaMemcpyDeviceToDevice, st));
    void* g0 = d->d_cls;
    void* g1 = d->d_bbox;
    {
    PScope ps_loss(d, P_LOSS, 0, 0, 4);
    LossArgs la{d->scale, d->losses, 0};
    if (!side) {
        CK(sigmoid_bce(d->dt, d->rpn_logits.p, static_cast<int64_t>(d->n_loc) * cf.batch, d->A, d->A_pad,
                       d->a_labels, d->d_rpn_logits, la, d->ws, st));
        la.slot = 1;
        CK(rpn_smooth_l1(d->dt, d->rpn_deltas.p, static_cast<int64_t>(d->n_loc) * cf.batch, d->A, d->A_pad,
                         d->a_labels, d->a_targets, 1.0 / 9.0, static_cast<double>(cf.rpn_batch) * cf.batch,
                         d->d_rpn_deltas, la, d->ws, st));
    }
    la.slot = 2;
    CK(softmax_ce(d->dt, d->cls_logits.p, d->R, d->ncls, d->ncls_pad, d->roi_labels, g0, la, d->ws, st));
    la.slot = 3;
    CK(rcnn_smooth_l1(d->dt, d->bbox_pred.p, d->R, d->nbox_pad, d->roi_labels, d->roi_targets, 1.0, g1, la, d->ws,
                      st));
    }

    // ---- backward
    Bwd B{d, 0, 0};
    B.side = d->side_wgrad && !d->prof.on;
    for (bool& bz : d->dzr_busy) bz = false;  // the previous step joined the side stream
    d->dzb_busy = false;
    // fc layers (bbox then cls: reverse pack order)
    void* dpool = d->gbuf[2];
    conv_wgrad_to(B, d->fc_bbox, d->pooled, g1);
    dgrad(d, d->fc_bbox, g1, dpool, 0);
    conv_wgrad_to(B, d->fc_cls, d->pooled, g0);
    dgrad(d, d->fc_cls, g0, dpool, 1);
    // avgpool, then the res5 head
    void* dhead = d->gbuf[3];
    void* cur = dhead;
    void* spare = d->gbuf[2];
    const float neg = cf.mode == 0 ? 0.0f : cf.slope;
    d->dpool_cur = dpool;
    if (!d->head_pool_bwd) {
        // avgpool backward with the last head block's output activation (its dS)
        // fused in; inner block boundaries are masked in the dgrad epilogues
        // (with head_pool_fuse the last block's bn3 backward forms dS itself)
        PScope ps(d, P_POOL, 0, static_cast<double>(d->es) * 2.0 * d->head_out.numel());
        CK(avgpool_bwd(d->dt, dpool, d->R, d->head_out.h * d->head_out.w, d->feat_c, dhead, st,
                       d->head.empty() || d->head_pool_fuse ? nullptr : d->head_out.p, neg,
                       d->head_pool_fuse ? d->head.back().obits : nullptr));
    }
    for (int i = static_cast<int>(d->head.size()) - 1; i >= 0; --i) {
        const void* in_mask = i > 0 ? d->head[i - 1].out.p : nullptr;  // head[0].in = RoIAlign output (linear)
        block_bwd(B, d->head[i], cur, spare, d->gbuf[1], d->gbuf[4], in_mask, i > 0 ? d->head[i - 1].obits : nullptr);
        std::swap(cur, spare);
    }
    (void)spare;
    // cur = d roi_feat
    void* dc4 = d->gbuf[(cur == d->gbuf[2]) ? 3 : 2];
    { PScope ps(d, P_ROI_B, 0, static_cast<double>(d->es) * (d->roi_feat.numel() + d->c4.numel()));
    CK(roialign_bwd(d->dt, cur, d->c4.n, d->c4.h, d->c4.w, d->c4.c, d->rois, d->R, d->P, sscale, cf.sampling_ratio,
                    dc4, d->ws, d->ws_bytes, st, d->roi_step)); }
    // RPN head backward (bbox, cls, conv)
    if (side) {
        // done on the side stream behind the proposal layer: only the rpn_conv
        // dgrad (onto the RoIAlign gradient, then the c4 activation mask) is left
        CK(cudaStreamWaitEvent(st, d->ev_rpn_join, 0));
        dgrad(d, d->rpn_conv, d->drpn_side, dc4, 1, nullptr, d->c4.p, neg,
              d->backbone.empty() ? nullptr : d->backbone.back().obits);
    } else {
    void* drpn = dz_buf(B, d->gbuf[0]);
    conv_wgrad_to(B, d->rpn_bbox, d->rpn_a, d->d_rpn_deltas);
    conv_wgrad_to(B, d->rpn_cls, d->rpn_a, d->d_rpn_logits);
    // the RPN ReLU backward is folded into whichever dgrad writes drpn last (the
    // one with K % 64 == 0 on the tensor-core path)
    const bool bbox_last = (d->rpn_bbox.g.K % 64) == 0 || d->dt != kF16;
    const ConvL& r_first = bbox_last ? d->rpn_cls : d->rpn_bbox;
    const ConvL& r_last = bbox_last ? d->rpn_bbox : d->rpn_cls;
    dgrad(d, r_first, bbox_last ? d->d_rpn_logits : d->d_rpn_deltas, drpn, 0);
    if ((r_last.g.K % 64) == 0 || d->dt != kF16) {
        dgrad(d, r_last, bbox_last ? d->d_rpn_deltas : d->d_rpn_logits, drpn, 1, nullptr, d->rpn_a.p, 0.0f);
    } else {
        dgrad(d, r_last, bbox_last ? d->d_rpn_deltas : d->d_rpn_logits, drpn, 1);
        PScope ps(d, P_ELEM, 0, 3.0 * d->es * d->rpn_a.numel());
        CK(act_bwd(d->dt, drpn, d->rpn_a.p, drpn, d->rpn_a.numel(), 0.0f, st));
    }
    conv_wgrad_to(B, d->rpn_conv, d->c4, drpn);
    // dc4 (RoIAlign part) + RPN part, then the last backbone block's activation mask
    dgrad(d, d->rpn_conv, drpn, dc4, 1, nullptr, d->c4.p, neg, d->backbone.empty() ? nullptr : d->backbone.back().obits);
    }
    // backbone
    cur = dc4;
    spare = dc4 == d->gbuf[2] ? d->gbuf[3] : d->gbuf[2];
    const int L = static_cast<int>(d->backbone.size());
    for (int i = L - 1; i >= 0; --i) {
        if (!d->ck_start.empty() && i + 1 < L) {
            const auto it = std::find(d->ck_start.begin(), d->ck_start.end(), i + 1);
            if (it != d->ck_start.end()) {
                // block i closes a segment that is not the last: refill the arena
                // from the segment's boundary input (src/memopt.cpp:183-189), once
                // the deferred wgrads of the segment above stopped reading it
                if (B.side) {
                    CK(cudaEventRecord(d->ck_ev, d->wst));
                    CK(cudaStreamWaitEvent(st, d->ck_ev, 0));
                }
                for (int j = *(it - 1); j <= i; ++j) block_fwd(d, d->backbone[j]);
            }
        }
        const void* in_mask = i > 0 ? d->backbone[i - 1].out.p : nullptr;  // backbone[0].in = max-pool output
        block_bwd(B, d->backbone[i], cur, spare, d->gbuf[1], d->gbuf[4], in_mask,
                  i > 0 ? d->backbone[i - 1].obits : nullptr);
        std::swap(cur, spare);
    }
    // maxpool, stem norm, stem wgrad (the image gradient is not needed)
    { PScope ps(d, P_POOL, 0, d->es * (2.0 * d->stem_a.numel() + d->pool.numel()));
    CK(maxpool_bwd(d->dt, cur, d->pool_arg, d->stem_a.n, d->stem_a.h, d->stem_a.w, d->stem_a.c, 3, 2, 1, spare, st)); }
    void* dstem = dz_buf(B, d->gbuf[0]);
    norm_bwd(d, d->stem_n, d->stem_z, d->stem_a, spare, dstem);
    if (d->stem_gemm) {
        // dW' = X'^T dZ as a 1x1 wgrad; folded back to [64][7][7][8] once reduced
        ConvL c2 = d->stem2;
        c2.p = d->stem.p;  // its arena slice / job
        stem_wgrad_to(B, c2, d->stem_x2, dstem);
    } else {
        conv_wgrad_to(B, d->stem, d->img, dstem);
    }
    if (B.side) {
        CK(cudaEventRecord(d->wev_join, d->wst));
        CK(cudaStreamWaitEvent(st, d->wev_join, 0));
    }

    if (d->defer_wgrad)
        for (int left : d->bucket_left)
            if (left != 0) throw std::runtime_error("gradient bucket left incomplete by the backward schedule");

    // ---- data-parallel reduction, overflow check, update
    if (d->comm_on) {
        if (!d->defer_wgrad) grads_ready(B, 0);  // flush any remaining bucket
        PScope ps(d, P_COMM, 0, 4.0 * d->n_bn + 32.0);
        CK(cudaEventRecord(d->ev_fork, st));
        CK(cudaStreamWaitEvent(d->comm, d->ev_fork, 0));
        CKC(comm_allreduce(d->ctx, d->bng, d->n_bn, kF32, 0, d->comm));
        CKC(comm_allreduce(d->ctx, d->losses, 4, 3 /* f64 */, 0, d->comm));
        // the reduces flagged this rank's fp16 gradients before the averaging
        // allreduce; an average of finite values is finite and a non-finite
        // input stays non-finite, so the summed gradient overflows iff some
        // rank flagged (MAX over ranks)
        if (d->defer_wgrad) CKC(comm_allreduce(d->ctx, d->flag, 1, 2 /* int32 */, 2 /* max */, d->comm));
        CK(cudaEventRecord(d->ev_join, d->comm));
        CK(cudaStreamWaitEvent(st, d->ev_join, 0));
    }
    // algorithmic bytes: gradient read, fp32 master + velocity read and written,
    // fp16 shadow written (20 B/param in fp16 mode); BN params 20 B (fp32 grads)
    PScope ps_opt(d, P_OPTIM, 0, (d->es + 16.0 + (d->dt == kF16 ? 2.0 : 0.0)) * d->n_w + 20.0 * d->n_bn, 5);
    if (!d->defer_wgrad) CK(nonfinite_check(d->dt, d->g, d->n_w, d->flag, st));  // else: in the reduces
    CK(nonfinite_check(kF32, d->bng, d->n_bn, d->flag, st));
    const double K = static_cast<double>(d->ctx->world);
    // fp16 buckets arrive averaged over the ranks (issue_bucket_allreduce)
    const double Kw = d->dt == kF16 ? 1.0 : K;
    if (d->shard) {
        // this rank's shard of every bucket, then the fp16 shadows all-gathered
        // on the comm stream (each bucket as soon as its shard is updated)
        const int64_t r = d->ctx->rank, Kr = d->ctx->world;
        for (size_t b = 0; b < d->buckets.size(); ++b) {
            const auto [lo, hi] = d->buckets[b];
            const int64_t cnt = (hi - lo) / Kr, s = lo + r * cnt;
            CK(fused_sgd(kF16, static_cast<__half*>(d->g) + s, d->w32 + s, d->v32 + s,
                         static_cast<__half*>(d->wdev) + s, cnt, cf.lr, cf.momentum, d->scale, Kw, d->flag, st));
            CK(cudaEventRecord(d->gather_ev[b], st));
            CK(cudaStreamWaitEvent(d->comm, d->gather_ev[b], 0));
            CKC(comm_all_gather(d->ctx, static_cast<__half*>(d->wdev) + lo, cnt, kF16, d->comm));
        }
        CK(cudaEventRecord(d->ev_gather_join, d->comm));
        CK(cudaStreamWaitEvent(st, d->ev_gather_join, 0));
        d->masters_synced = Kr == 1;
    } else {
        CK(fused_sgd(d->dt, d->g, d->w32, d->v32, d->dt == kF16 ? static_cast<__half*>(d->wdev) : nullptr, d->n_w,
                     cf.lr, cf.momentum, d->scale, Kw, d->flag, st));
    }
    CK(fused_sgd(kF32, d->bng, d->bn32, d->bnv, nullptr, d->n_bn, cf.lr, cf.momentum, d->scale, K, d->flag, st));
    CK(update_scale_device(d->scale, d->good, d->flag, cf.dynamic_scale, cf.growth_interval, cf.growth, cf.backoff,
                           cf.min_scale, cf.max_scale, st));
}

}  // namespace

// ====================================================================== ABI
extern "C" {

int sdb_plan_buckets(const int64_t* offsets, int n, int64_t total, int64_t cap_elems, int64_t* out_lo_hi, int cap_out) {
    // gradient buckets over the flat buffer, formed from the END because the
    // backward pass completes the last layers first; a bucket closes at the
    // first parameter boundary where it reaches cap_elems (the first
    // parameter always closes the last bucket)
    int nb = 0;
    int64_t hi = total;
    for (int i = n - 1; i >= 0; --i) {
        if (hi - offsets[i] >= cap_elems || i == 0) {
            if (nb < cap_out) {
                out_lo_hi[2 * nb] = offsets[i];
                out_lo_hi[2 * nb + 1] = hi;
            }
            ++nb;
            hi = offsets[i];
        }
    }
    if (hi > 0) {
        if (nb < cap_out) {
            out_lo_hi[2 * nb] = 0;
            out_lo_hi[2 * nb + 1] = hi;
        }
        ++nb;
    }
    return nb;
}

int sdb_det_create(sdb_ctx* ctx, const sdb_det_config* cfgp, sdb_det** out) {
    if (!ctx || !cfgp || !out) return det_fail(SDB_PARAM, "null argument");
    const sdb_det_config& cf = *cfgp;
    if (cf.batch < 1 || cf.img_h < 32 || cf.img_w < 32) return det_fail(SDB_SHAPE, "bad batch/image size");
    if (cf.mode < 0 || cf.mode > 2) return det_fail(SDB_PARAM, "mode must be 0 (fp32/BN), 1 (fp16/IABN), 2 (fp32/IABN)");
    if (cf.n_scales < 1 || cf.n_scales > 8 || cf.n_ratios < 1 || cf.n_ratios > 8) return det_fail(SDB_PARAM, "anchors");
    if (cf.nms_iou < 0.0 || cf.nms_iou > 1.0) return det_fail(SDB_PARAM, "iou threshold outside [0,1]");
    if (cf.mode >= 1 && !(cf.slope > 0.0f)) return det_fail(SDB_NONINVERTIBLE, "iabn requires slope > 0");
    if (cf.sync_bn && cf.mode != 0) return det_fail(SDB_PARAM, "sync_bn is a BN mode (mode 0); IABN statistics stay per GPU");
    auto* d = new sdb_det();
    try {
        d->ctx = ctx;
        d->cfg = cf;
        d->dt = cf.mode == 1 ? kF16 : kF32;
        d->es = cf.mode == 1 ? 2 : 4;
        d->use_graph = std::getenv("SDB_NO_GRAPH") == nullptr;
        CK(cudaSetDevice(ctx->device));
        const int b = cf.batch;
        // ---- parameters (reference pack order)
        d->stem = d->conv("stem.conv", 3, 64, 7, 2, 3);
        d->params[d->stem.p].C = 8;  // input channels padded 3 -> 8 on device (16-byte rows)
        d->n_w = d->params[d->stem.p].off + 64 * 7 * 7 * 8;
        d->params[d->stem.p].numel = 64 * 7 * 7 * 8;
        d->stem.g.C = 8;
        d->stem_n = d->norm("stem.bn", 64, true, false);
        build_stage(d, d->backbone, "res2", cf.blocks[0], 64, 64, 256, 1);
        build_stage(d, d->backbone, "res3", cf.blocks[1], 256, 128, 512, 2);
        build_stage(d, d->backbone, "res4", cf.blocks[2], 512, 256, 1024, 2);
        d->A = cf.n_scales * cf.n_ratios;
        d->A_pad = round_up(d->A, 8);
        d->rpn_conv = d->conv("rpn.conv", 1024, cf.rpn_channels, 3, 1, 1);
        {
            const int pc = d->add_param("rpn.cls", {d->A, cf.rpn_channels, 1, 1}, 0, d->A_pad, 1, 1, cf.rpn_channels);
            d->rpn_cls.p = pc;
            d->rpn_cls.g = ConvShape{0, 0, 0, cf.rpn_channels, d->A_pad, 1, 1, 1, 0};
            const int pb = d->add_param("rpn.bbox", {4 * d->A, cf.rpn_channels, 1, 1}, 0, 4 * d->A_pad, 1, 1,
                                        cf.rpn_channels);
            d->rpn_bbox.p = pb;
            d->rpn_bbox.g = ConvShape{0, 0, 0, cf.rpn_channels, 4 * d->A_pad, 1, 1, 1, 0};
        }
        d->feat_c = 1024;
        if (cf.blocks[3] > 0) {
            build_stage(d, d->head, "res5", cf.blocks[3], 1024, 512, 2048, 2);
            d->feat_c = 2048;
        }
        d->ncls = cf.num_classes + 1;
        d->ncls_pad = round_up(d->ncls, 8);
        d->nbox_pad = round_up(4 * d->ncls, 8);
        d->fc_cls.p = d->add_param("fc.cls", {d->feat_c, d->ncls}, 1, d->ncls_pad, 1, 1, d->feat_c);
        d->fc_bbox.p = d->add_param("fc.bbox", {d->feat_c, 4 * d->ncls}, 1, d->nbox_pad, 1, 1, d->feat_c);

        // ---- activations
        d->img = d->act(b, cf.img_h, cf.img_w, 8);
        d->stem.g.N = b; d->stem.g.H = cf.img_h; d->stem.g.W = cf.img_w;
        d->stem_z = d->act(b, d->stem.g.Ho(), d->stem.g.Wo(), 64);
        d->stem_gemm = d->dt == kF16 && std::getenv("SDB_NO_STEM_GEMM") == nullptr;
        if (d->stem_gemm) {
            const int64_t px = d->stem_z.numel() / 64;
            d->stem2.p = d->stem.p;
            d->stem2.g = ConvShape{1, 1, static_cast<int>(px), 192, 64, 1, 1, 1, 0};
            d->stem_x2 = d->alloc(static_cast<size_t>(px) * 192 * 2);
            d->stem_w2 = d->alloc(64 * 192 * 2);
            d->stem_dw2 = d->alloc(64 * 192 * 2);
        }
        d->stem_a = cf.mode == 0 ? d->act(b, d->stem_z.h, d->stem_z.w, 64) : d->stem_z;
        const int ph = (d->stem_a.h + 2 - 3) / 2 + 1, pw = (d->stem_a.w + 2 - 3) / 2 + 1;
        d->pool = d->act(b, ph, pw, 64);
        d->pool_arg = static_cast<uint8_t*>(d->alloc(static_cast<size_t>(d->pool.numel())));
        d->gbuf_elems = std::max(d->stem_z.numel(), d->pool.numel());
        if (cf.checkpoint) {
            // sizing pass (no allocation), then the arena, then the real pass
            d->ck_start = plan_segments(static_cast<int>(d->backbone.size()));
            d->measuring = true;
            alloc_stage(d, d->backbone, d->pool, d->ck_start);
            d->measuring = false;
            d->bytes_backbone = 0;
            d->ck_arena = static_cast<uint8_t*>(d->alloc(d->ck_bytes));
            alloc_stage(d, d->backbone, d->pool, d->ck_start);
            d->bytes_backbone += static_cast<int64_t>(d->ck_bytes);
            CK(cudaEventCreateWithFlags(&d->ck_ev, cudaEventDisableTiming));
        } else {
            alloc_stage(d, d->backbone, d->pool);
        }
        d->c4 = d->backbone.back().out;
        d->fh = d->c4.h;
        d->fw = d->c4.w;
        d->n_loc = d->fh * d->fw;
        d->nA = d->n_loc * d->A;
        auto setg = [](ConvL& c, const Act& x) { c.g.N = x.n; c.g.H = x.h; c.g.W = x.w; };
        setg(d->rpn_conv, d->c4);
        d->rpn_z = d->act(b, d->fh, d->fw, cf.rpn_channels);
        d->rpn_a = d->act(b, d->fh, d->fw, cf.rpn_channels);
        setg(d->rpn_cls, d->rpn_a);
        setg(d->rpn_bbox, d->rpn_a);
        d->rpn_logits = d->act(b, d->fh, d->fw, d->A_pad);
        d->rpn_deltas = d->act(b, d->fh, d->fw, 4 * d->A_pad);
        d->R = b * cf.roi_batch;
        d->P = cf.pool;
        // The res5 entry block reads the RoIAlign output only through 1x1
        // stride-2 pad-0 convolutions (conv1 and the shortcut), i.e. only the
        // even bins.  Pool just those bins (bitwise the same values) and run
        // both convolutions at stride 1: 3/4 of the RoIAlign output, its
        // gradient and the dgrad zero phases are never materialised.
        if (!d->head.empty() && d->P % 2 == 0) {
            Block& h0 = d->head[0];
            auto one_by_one_s2 = [](const ConvL& c) { return c.g.R == 1 && c.g.S == 1 && c.g.stride == 2 && c.g.pad == 0; };
            if (one_by_one_s2(h0.c1) && h0.has_down && one_by_one_s2(h0.down)) {
                d->roi_step = 2;
                h0.c1.g.stride = 1;
                h0.down.g.stride = 1;
            }
        }
        const int Po = (d->P + d->roi_step - 1) / d->roi_step;
        d->roi_feat = d->act(d->R, Po, Po, 1024);
        d->gbuf_elems = std::max({d->gbuf_elems, d->c4.numel(), d->rpn_z.numel(), d->roi_feat.numel(),
                                  d->rpn_deltas.numel()});
        if (!d->head.empty()) {
            alloc_stage(d, d->head, d->roi_feat);
            d->head_out = d->head.back().out;
        } else {
            d->head_out = d->roi_feat;
        }
        d->pooled = d->act(d->R, 1, 1, d->feat_c);
        d->head_pool_fuse = !d->head.empty() && d->dt == kF16 && cf.mode == 1 && d->head.back().n3.act == 2 &&
                            d->head.back().obits != nullptr && d->feat_c == 2048 &&
                            std::getenv("SDB_NO_HEAD_POOL_FUSE") == nullptr;
        d->head_pool_bwd = d->head_pool_fuse && !d->head.back().has_down &&
                           std::getenv("SDB_NO_HEAD_POOL_BWD") == nullptr;
        setg(d->fc_cls, d->pooled);
        setg(d->fc_bbox, d->pooled);
        d->fc_cls.g.C = d->feat_c; d->fc_cls.g.K = d->ncls_pad; d->fc_cls.g.R = d->fc_cls.g.S = 1;
        d->fc_cls.g.stride = 1; d->fc_cls.g.pad = 0;
        d->fc_bbox.g = d->fc_cls.g;
        d->fc_bbox.g.K = d->nbox_pad;
        d->cls_logits = d->act(d->R, 1, 1, d->ncls_pad);
        d->bbox_pred = d->act(d->R, 1, 1, d->nbox_pad);
        d->gbuf_elems = std::max({d->gbuf_elems, d->head_out.numel(), d->bbox_pred.numel()});
        for (auto& gb : d->gbuf) gb = d->alloc(static_cast<size_t>(d->gbuf_elems) * d->es);
        d->d_rpn_logits = d->alloc(static_cast<size_t>(d->rpn_logits.numel()) * d->es);
        d->d_rpn_deltas = d->alloc(static_cast<size_t>(d->rpn_deltas.numel()) * d->es);
        d->d_cls = d->alloc(static_cast<size_t>(d->cls_logits.numel()) * d->es);
        d->d_bbox = d->alloc(static_cast<size_t>(d->bbox_pred.numel()) * d->es);

        // ---- parameter state
        d->w32 = static_cast<float*>(d->alloc(d->n_w * 4));
        d->v32 = static_cast<float*>(d->alloc(d->n_w * 4));
        d->wdev = cf.mode == 1 ? d->alloc(d->n_w * 2) : d->w32;
        d->g = d->alloc(d->n_w * d->es);
        CK(cudaMemset(d->g, 0, d->n_w * d->es));
        d->bn32 = static_cast<float*>(d->alloc(d->n_bn * 4));
        d->bnv = static_cast<float*>(d->alloc(d->n_bn * 4));
        d->bng = static_cast<float*>(d->alloc(d->n_bn * 4));
        d->scale = static_cast<double*>(d->alloc(8));
        d->good = static_cast<int64_t*>(d->alloc(8));
        d->flag = static_cast<int*>(d->alloc(4));
        d->losses = static_cast<double*>(d->alloc(8 * 8));
        d->scale_used = static_cast<double*>(d->alloc(8));
        const double s0 = cf.mode == 1 ? cf.scale_init : 1.0;
        const int64_t zero = 0;
        CK(cudaMemcpyAsync(d->scale, &s0, 8, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(d->good, &zero, 8, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemsetAsync(d->losses, 0, 64, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));

        // ---- targets / proposals buffers
        d->anchors = static_cast<float*>(d->alloc(static_cast<size_t>(d->nA) * 16));
        AnchorCfg ac{};
        ac.H = d->fh; ac.W = d->fw; ac.stride = 16.0f; ac.ns = cf.n_scales; ac.nr = cf.n_ratios;
        for (int i = 0; i < cf.n_scales; ++i) ac.scales[i] = cf.scales[i];
        for (int i = 0; i < cf.n_ratios; ++i) ac.ratios[i] = cf.ratios[i];
        CK(make_anchors(ac, d->anchors, ctx->stream));
        d->gt = static_cast<float*>(d->alloc(static_cast<size_t>(b) * cf.max_gt * 16));
        d->gt_cls = static_cast<int32_t*>(d->alloc(static_cast<size_t>(b) * cf.max_gt * 4));
        d->gt_count = static_cast<int32_t*>(d->alloc(b * 4));
        d->keys = static_cast<uint64_t*>(d->alloc(2 * b * 8));
        d->a_labels = static_cast<int8_t*>(d->alloc(static_cast<size_t>(b) * d->nA));
        d->a_targets = static_cast<float*>(d->alloc(static_cast<size_t>(b) * d->nA * 16));
        d->props = static_cast<float*>(d->alloc(static_cast<size_t>(b) * cf.post_nms * 16));
        d->prop_count = static_cast<int32_t*>(d->alloc(b * 4));
        d->keep_pos = static_cast<int32_t*>(d->alloc(static_cast<size_t>(b) * cf.post_nms * 4));
        const int ws_stride = cf.post_nms + cf.max_gt;
        d->pt_flag = static_cast<int8_t*>(d->alloc(static_cast<size_t>(b) * ws_stride));
        d->pt_arg = static_cast<int32_t*>(d->alloc(static_cast<size_t>(b) * ws_stride * 4));
        d->rois = static_cast<float*>(d->alloc(static_cast<size_t>(d->R) * 20));
        d->roi_labels = static_cast<int32_t*>(d->alloc(static_cast<size_t>(d->R) * 4));
        d->roi_targets = static_cast<float*>(d->alloc(static_cast<size_t>(d->R) * 16));
        d->roi_count = static_cast<int32_t*>(d->alloc(b * 4));
        d->ws_bytes = max_ws(d);
        d->ws = d->alloc(d->ws_bytes);
        if (cf.sync_bn) d->sbn_red = static_cast<float*>(d->alloc(2 * 2048 * sizeof(float)));
        if (d->dt == kF16) {
            d->cst.cap_bytes = static_cast<size_t>(2 * 148) * 4 * 2 * 256 * sizeof(double);  // 2 CTAs x 148 SMs
            d->cst.buf = static_cast<double*>(d->alloc(d->cst.cap_bytes));
            if (cf.mode == 1) {
                d->cst_b.cap_bytes = d->cst.cap_bytes;
                d->cst_b.buf = static_cast<double*>(d->alloc(d->cst_b.cap_bytes));
            }
        }
        d->comm_on = ctx->nccl != nullptr;
        d->defer_wgrad = d->dt == kF16 && std::getenv("SDB_NO_DEFER_WGRAD") == nullptr;
        if (d->defer_wgrad) {
            size_t off = 0;
            auto add = [&](const ConvL& c) {
                if (c.p < 0 || d->wg_off.count(c.p)) return;
                d->wg_off[c.p] = off;
                off += (conv_wgrad_workspace(c.g, d->dt) + 255) & ~size_t(255);
            };
            add(d->stem_gemm ? d->stem2 : d->stem);
            for (auto* stg : {&d->backbone, &d->head})
                for (auto& bl : *stg) {
                    add(bl.c1); add(bl.c2); add(bl.c3);
                    if (bl.has_down) add(bl.down);
                }
            add(d->rpn_conv); add(d->rpn_cls); add(d->rpn_bbox); add(d->fc_cls); add(d->fc_bbox);
            d->wg_arena = static_cast<uint8_t*>(d->alloc(off));
            d->side_wgrad = std::getenv("SDB_NO_SIDE_WGRAD") == nullptr;
        }
        if (d->dt == kF16 && cf.mode == 1 && std::getenv("SDB_NO_BRANCH") == nullptr) {
            int lo = 0, hi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CK(cudaStreamCreateWithPriority(&d->bst, cudaStreamNonBlocking, hi));
            CK(cudaEventCreateWithFlags(&d->ev_b_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&d->ev_b_join, cudaEventDisableTiming));
            d->cst2.cap_bytes = d->cst.cap_bytes;
            d->cst2.buf = static_cast<double*>(d->alloc(d->cst2.cap_bytes));
            size_t m2 = 0;
            for (auto& bl : d->backbone)
                if (bl.has_down) m2 = std::max(m2, norm_workspace_bytes(static_cast<int64_t>(bl.zd.n) * bl.zd.h * bl.zd.w, bl.zd.c));
            for (auto& bl : d->head)
                if (bl.has_down) m2 = std::max(m2, norm_workspace_bytes(static_cast<int64_t>(bl.zd.n) * bl.zd.h * bl.zd.w, bl.zd.c));
            d->ws2 = d->alloc(std::max<size_t>(m2, 256));
            int64_t zmax = 0;
            for (auto& bl : d->backbone)
                if (bl.has_down) zmax = std::max(zmax, bl.zd.numel());
            for (auto& bl : d->head)
                if (bl.has_down) zmax = std::max(zmax, bl.zd.numel());
            if (std::getenv("SDB_NO_BRANCH_BWD") == nullptr) {
                d->dzb = d->alloc(static_cast<size_t>(std::max<int64_t>(zmax, 1)) * d->es);
                CK(cudaEventCreateWithFlags(&d->ev_b2_fork, cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&d->ev_dzb, cudaEventDisableTiming));
            }
        }
        if (d->side_wgrad) {
            int lo = 0, hi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            // lower priority than the main stream's dgrad/norm chain (the critical path)
            CK(cudaStreamCreateWithPriority(&d->wst, cudaStreamNonBlocking, lo));
            CK(cudaEventCreateWithFlags(&d->wev_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&d->wev_join, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&d->ev_at_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&d->ev_at_join, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&d->ev_rpn_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&d->ev_rpn_join, cudaEventDisableTiming));
            d->drpn_side = d->alloc(static_cast<size_t>(d->rpn_a.numel()) * d->es);
            d->ws_at = d->alloc(anchor_target_workspace_bytes(cf.batch, d->nA, cf.max_gt));
            if (const char* e = std::getenv("SDB_DZ_RING")) d->dzr_n = std::max(2, std::min(sdb_det::kDzRing, std::atoi(e)));
            for (int k = 0; k < d->dzr_n; ++k) {
                d->dzr[k] = d->alloc(static_cast<size_t>(d->gbuf_elems) * d->es);
                CK(cudaEventCreateWithFlags(&d->dzr_ev[k], cudaEventDisableTiming));
            }
        }
        for (int k = 0; k < sdb_det::kStage; ++k) {
            CK(cudaMallocHost(&d->h_gt[k], static_cast<size_t>(b) * cf.max_gt * 16));
            CK(cudaMallocHost(&d->h_cls[k], static_cast<size_t>(b) * cf.max_gt * 4));
            CK(cudaMallocHost(&d->h_cnt[k], b * 4));
            CK(cudaMallocHost(&d->h_keys[k], 2 * b * 8));
            CK(cudaMallocHost(&d->h_slots[k], b * 8));
            CK(cudaEventCreateWithFlags(&d->stage_ev[k], cudaEventDisableTiming));
        }
        d->slots_dev = static_cast<int64_t*>(d->alloc(b * 8));
        CK(cudaMallocHost(&d->h_losses, 16 * 8));

        // ---- gradient buckets over the flat fp16/fp32 gradient, formed from the
        // END (backward produces the last layers first); planned at every world
        // size, so one schedule serves N = 1 and N > 1
        if (d->comm_on || d->defer_wgrad) {
            const int64_t cap = static_cast<int64_t>(cf.bucket_mb * 1024 * 1024 / d->es);
            std::vector<int64_t> offs;
            for (const Param& p : d->params)
                if (p.kind <= 1) offs.push_back(p.off);
            std::vector<int64_t> lohi(2 * offs.size() + 2);
            const int nb = sdb_plan_buckets(offs.data(), static_cast<int>(offs.size()), d->n_w, cap, lohi.data(),
                                            static_cast<int>(offs.size()) + 1);
            for (int i = 0; i < nb; ++i) d->buckets.push_back({lohi[2 * i], lohi[2 * i + 1]});
            d->bucket_of.assign(d->params.size(), -1);
            d->bucket_nparams.assign(d->buckets.size(), 0);
            for (size_t pi = 0; pi < d->params.size(); ++pi) {
                if (d->params[pi].kind > 1) continue;
                for (size_t bi = 0; bi < d->buckets.size(); ++bi)
                    if (d->params[pi].off >= d->buckets[bi].first && d->params[pi].off < d->buckets[bi].second) {
                        d->bucket_of[pi] = static_cast<int>(bi);
                        ++d->bucket_nparams[bi];
                    }
            }
            d->bjobs.resize(d->buckets.size());
            d->btab.resize(d->buckets.size());
            for (size_t i = 0; i < d->buckets.size(); ++i) {
                cudaEvent_t e;
                CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                d->bucket_ev.push_back(e);
            }
        }
        if (d->comm_on) {
            int plo = 0, phi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&plo, &phi));
            CK(cudaStreamCreateWithPriority(&d->comm, cudaStreamNonBlocking, phi));
            CK(cudaEventCreateWithFlags(&d->ev_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&d->ev_join, cudaEventDisableTiming));
            // the sharded update needs every bucket to split evenly over the ranks
            bool even = true;
            for (const auto& bk : d->buckets) even = even && (bk.second - bk.first) % ctx->world == 0;
            d->shard = d->defer_wgrad && cf.shard_optimizer && even;
            if (d->shard) {
                for (size_t i = 0; i < d->buckets.size(); ++i) {
                    cudaEvent_t e;
                    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                    d->gather_ev.push_back(e);
                }
                CK(cudaEventCreateWithFlags(&d->ev_gather_join, cudaEventDisableTiming));
            }
        }
        init_params(d);
    } catch (const std::exception& e) {
        for (void* p : d->allocs) cudaFree(p);
        delete d;
        return det_fail(SDB_CUDA, e.what());
    }
    *out = d;
    return SDB_OK;
}

int sdb_det_destroy(sdb_det* d) {
    if (!d) return SDB_OK;
    cudaStreamSynchronize(d->ctx->stream);
    if (d->gexec) cudaGraphExecDestroy(d->gexec);
    for (void* p : d->allocs) cudaFree(p);
    for (int k = 0; k < sdb_det::kStage; ++k) {
        cudaFreeHost(d->h_gt[k]);
        cudaFreeHost(d->h_cls[k]);
        cudaFreeHost(d->h_cnt[k]);
        cudaFreeHost(d->h_keys[k]);
        cudaFreeHost(d->h_slots[k]);
        if (d->stage_ev[k]) cudaEventDestroy(d->stage_ev[k]);
    }
    cudaFreeHost(d->h_losses);
    if (d->ck_ev) cudaEventDestroy(d->ck_ev);
    if (d->bst) {
        cudaEventDestroy(d->ev_b_fork);
        cudaEventDestroy(d->ev_b_join);
        if (d->ev_b2_fork) cudaEventDestroy(d->ev_b2_fork);
        if (d->ev_dzb) cudaEventDestroy(d->ev_dzb);
        cudaStreamDestroy(d->bst);
    }
    for (auto e : d->bucket_ev) cudaEventDestroy(e);
    if (d->wst) {
        for (auto e : d->dzr_ev)
            if (e) cudaEventDestroy(e);
        cudaEventDestroy(d->wev_fork);
        cudaEventDestroy(d->wev_join);
        cudaEventDestroy(d->ev_at_fork);
        cudaEventDestroy(d->ev_at_join);
        cudaEventDestroy(d->ev_rpn_fork);
        cudaEventDestroy(d->ev_rpn_join);
        cudaStreamDestroy(d->wst);
    }
    if (d->comm) {
        cudaEventDestroy(d->ev_fork);
        cudaEventDestroy(d->ev_join);
        for (auto e : d->gather_ev) cudaEventDestroy(e);
        if (d->ev_gather_join) cudaEventDestroy(d->ev_gather_join);
        cudaStreamDestroy(d->comm);
    }
    delete d;
    return SDB_OK;
}

int sdb_det_num_params(sdb_det* d, int* n_tensors, int64_t* n_w, int64_t* n_bn) {
    if (n_tensors) *n_tensors = static_cast<int>(d->params.size());
    if (n_w) *n_w = d->n_w;
    if (n_bn) *n_bn = d->n_bn;
    return SDB_OK;
}

int sdb_det_param_info(sdb_det* d, int idx, char* name, int name_len, int64_t* shape4, int* ndim, int* kind) {
    if (idx < 0 || idx >= static_cast<int>(d->params.size())) return det_fail(SDB_PARAM, "param index");
    const Param& p = d->params[idx];
    if (name && name_len > 0) {
        std::strncpy(name, p.name.c_str(), name_len - 1);
        name[name_len - 1] = 0;
    }
    if (ndim) *ndim = static_cast<int>(p.ref_shape.size());
    if (shape4)
        for (size_t i = 0; i < 4; ++i) shape4[i] = i < p.ref_shape.size() ? p.ref_shape[i] : 1;
    if (kind) *kind = p.kind;
    return SDB_OK;
}

// with the sharded optimizer each rank updated only its shard of the fp32
// masters and velocity: gather the full arrays once before host reads
static void sync_masters(sdb_det* d) {
    if (d->masters_synced) return;
    cudaStream_t st = d->ctx->stream;
    const int64_t Kr = d->ctx->world;
    for (const auto& bk : d->buckets) {
        const int64_t cnt = (bk.second - bk.first) / Kr;
        CKC(comm_all_gather(d->ctx, d->w32 + bk.first, cnt, kF32, st));
        CKC(comm_all_gather(d->ctx, d->v32 + bk.first, cnt, kF32, st));
    }
    CK(cudaStreamSynchronize(st));
    d->masters_synced = true;
}

// which: 0 get w, 1 set w, 2 get grad, 3 get velocity, 4 set velocity
static int param_xfer(sdb_det* d, int idx, float* host, int which) {
    if (idx < 0 || idx >= static_cast<int>(d->params.size())) return det_fail(SDB_PARAM, "param index");
    const Param& p = d->params[idx];
    cudaStream_t st = d->ctx->stream;
    try {
        if (which != 2 && p.kind <= 1) sync_masters(d);
        // every copy is ordered on the context stream: a pageable cudaMemcpy may
        // return before its DMA lands, and the stream is non-blocking
        CK(cudaStreamSynchronize(st));
        if (p.kind >= 2) {
            float* src = (which == 2 ? d->bng : (which >= 3 ? d->bnv : d->bn32)) + p.off;
            if (which == 1 || which == 4) CK(cudaMemcpyAsync(src, host, p.numel * 4, cudaMemcpyHostToDevice, st));
            else CK(cudaMemcpyAsync(host, src, p.numel * 4, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            return SDB_OK;
        }
        std::vector<float> dev(static_cast<size_t>(p.numel));
        if (which == 2) {
            if (d->dt == kF16) {
                std::vector<__half> h(static_cast<size_t>(p.numel));
                CK(cudaMemcpyAsync(h.data(), d->gptr(idx), p.numel * 2, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                for (size_t i = 0; i < h.size(); ++i) dev[i] = __half2float(h[i]);
            } else {
                CK(cudaMemcpyAsync(dev.data(), d->gptr(idx), p.numel * 4, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
            }
        } else {
            const float* src = which >= 3 ? d->v32 + p.off : d->wptr(idx);
            CK(cudaMemcpyAsync(dev.data(), src, p.numel * 4, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        }
        int64_t n = 1;
        for (int64_t s : p.ref_shape) n *= s;
        std::vector<float> ref(static_cast<size_t>(n));
        auto map = [&](auto fn) {
            if (p.kind == 0) {
                const int64_t O = p.ref_shape[0], Ci = p.ref_shape[1], kh = p.ref_shape[2], kw = p.ref_shape[3];
                for (int64_t o = 0; o < O; ++o)
                    for (int64_t c = 0; c < Ci; ++c)
                        for (int64_t r = 0; r < kh; ++r)
                            for (int64_t q = 0; q < kw; ++q)
                                fn(((o * Ci + c) * kh + r) * kw + q, ((o * p.R + r) * p.S + q) * p.C + c);
            } else {
                const int64_t in = p.ref_shape[0], outc = p.ref_shape[1];
                for (int64_t i = 0; i < in; ++i)
                    for (int64_t o = 0; o < outc; ++o) fn(i * outc + o, o * p.C + i);
            }
        };
        if (which == 1 || which == 4) {
            map([&](int64_t ri, int64_t di) { dev[di] = host[ri]; });
            CK(cudaMemcpyAsync(which == 4 ? d->v32 + p.off : d->wptr(idx), dev.data(), p.numel * 4,
                               cudaMemcpyHostToDevice, st));
            if (which == 1 && d->dt == kF16) CK(cast_f32_f16(d->wptr(idx), static_cast<__half*>(d->wdev_ptr(idx)), p.numel, st));
            CK(cudaStreamSynchronize(st));
        } else {
            map([&](int64_t ri, int64_t di) { host[ri] = dev[di]; });
        }
    } catch (const CollectiveFailure& e) {
        return det_fail(SDB_COLLECTIVE, e.what());
    } catch (const std::exception& e) {
        return det_fail(SDB_CUDA, e.what());
    }
    return SDB_OK;
}

int sdb_det_get_param(sdb_det* d, int idx, float* host) { return param_xfer(d, idx, host, 0); }
int sdb_det_set_param(sdb_det* d, int idx, const float* host) { return param_xfer(d, idx, const_cast<float*>(host), 1); }
int sdb_det_get_grad(sdb_det* d, int idx, float* host) { return param_xfer(d, idx, host, 2); }
int sdb_det_get_velocity(sdb_det* d, int idx, float* host) { return param_xfer(d, idx, host, 3); }
int sdb_det_set_velocity(sdb_det* d, int idx, const float* host) {
    return param_xfer(d, idx, const_cast<float*>(host), 4);
}

// ---- SDCK v1 checkpoints (src/checkpoint.cpp:47-128, little endian)
static int save_checkpoint_impl(sdb_det* d, const char* path, uint64_t config_digest, int64_t step) {
    std::ofstream f(path ? path : "", std::ios::binary);
    if (!f) return det_fail(SDB_FORMAT, "cannot open checkpoint for writing");
    auto bytes = [&](const void* p, size_t n) { f.write(static_cast<const char*>(p), static_cast<std::streamsize>(n)); };
    auto pod = [&](auto v) { bytes(&v, sizeof v); };
    bytes("SDCK", 4);
    pod(static_cast<uint32_t>(1));
    pod(config_digest);
    pod(step);
    pod(static_cast<uint32_t>(d->params.size()));
    std::vector<float> vel;
    for (int i = 0; i < static_cast<int>(d->params.size()); ++i) {
        const Param& p = d->params[i];
        int64_t n = 1;
        for (int64_t s2 : p.ref_shape) n *= s2;
        std::vector<float> w(static_cast<size_t>(n)), v(static_cast<size_t>(n));
        if (int rc = param_xfer(d, i, w.data(), 0)) return rc;
        if (int rc = param_xfer(d, i, v.data(), 3)) return rc;
        pod(static_cast<uint16_t>(p.name.size()));
        bytes(p.name.data(), p.name.size());
        pod(static_cast<uint8_t>(0));  // DType::F32 masters
        pod(static_cast<uint8_t>(p.ref_shape.size()));
        for (int64_t dim : p.ref_shape) pod(dim);
        bytes(w.data(), w.size() * sizeof(float));
        vel.insert(vel.end(), v.begin(), v.end());
    }
    pod(static_cast<uint64_t>(vel.size()));
    bytes(vel.data(), vel.size() * sizeof(float));
    double scale = 0.0;
    int64_t good = 0;
    try {
        CK(cudaMemcpyAsync(&scale, d->scale, 8, cudaMemcpyDeviceToHost, d->ctx->stream));
        CK(cudaMemcpyAsync(&good, d->good, 8, cudaMemcpyDeviceToHost, d->ctx->stream));
        CK(cudaStreamSynchronize(d->ctx->stream));
    } catch (const std::exception& e) {
        return det_fail(SDB_CUDA, e.what());
    }
    const auto& cf = d->cfg;
    pod(scale);
    pod(good);
    pod(static_cast<uint8_t>(cf.dynamic_scale ? 1 : 0));  // ScaleMode {Static, Dynamic}
    pod(static_cast<int64_t>(cf.growth_interval));
    pod(cf.growth);
    pod(cf.backoff);
    pod(cf.min_scale);
    pod(cf.max_scale);
    pod(static_cast<uint32_t>(0));  // running-stat blocks
    if (!f) return det_fail(SDB_FORMAT, "checkpoint write failed");
    return SDB_OK;
}

int sdb_det_save_checkpoint(sdb_det* d, const char* path, uint64_t config_digest, int64_t step) {
    try {
        return save_checkpoint_impl(d, path, config_digest, step);
    } catch (const std::exception& e) {
        return det_fail(SDB_FORMAT, std::string("checkpoint: ") + e.what());
    }
}

static int load_checkpoint_impl(sdb_det* d, const char* path, uint64_t* config_digest, int64_t* step) {
    std::ifstream f(path ? path : "", std::ios::binary);
    if (!f) return det_fail(SDB_FORMAT, "cannot open checkpoint");
    bool ok = true;
    auto bytes = [&](void* p, size_t n) {
        f.read(static_cast<char*>(p), static_cast<std::streamsize>(n));
        if (static_cast<size_t>(f.gcount()) != n) ok = false;
    };
    auto pod = [&](auto& v) { bytes(&v, sizeof v); };
    char magic[4];
    bytes(magic, 4);
    if (!ok || std::memcmp(magic, "SDCK", 4) != 0) return det_fail(SDB_FORMAT, "not a checkpoint file (bad magic)");
    uint32_t version = 0;
    pod(version);
    if (!ok || version != 1) return det_fail(SDB_FORMAT, "unsupported checkpoint version");
    uint64_t digest = 0;
    int64_t st = 0;
    uint32_t np = 0;
    pod(digest);
    pod(st);
    pod(np);
    if (!ok) return det_fail(SDB_FORMAT, "truncated checkpoint file");
    if (np != d->params.size()) return det_fail(SDB_CONTRACT, "checkpoint parameter count differs from this detector");
    std::vector<std::vector<float>> ws(np);
    for (uint32_t i = 0; i < np; ++i) {
        const Param& p = d->params[i];
        uint16_t len = 0;
        pod(len);
        std::string name(len, '\0');
        bytes(name.data(), len);
        uint8_t dtype = 0, rank = 0;
        pod(dtype);
        pod(rank);
        if (!ok) return det_fail(SDB_FORMAT, "truncated checkpoint file");
        if (rank < 1 || rank > 4) return det_fail(SDB_FORMAT, "checkpoint parameter rank out of range");
        std::vector<int64_t> shape(rank);
        for (auto& dim : shape) pod(dim);
        if (!ok) return det_fail(SDB_FORMAT, "truncated checkpoint file");
        if (name != p.name || shape != p.ref_shape || dtype != 0)
            return det_fail(SDB_CONTRACT, ("checkpoint parameter mismatch at " + p.name).c_str());
        int64_t n = 1;
        for (int64_t dim : shape) n *= dim;
        ws[i].resize(static_cast<size_t>(n));
        bytes(ws[i].data(), ws[i].size() * sizeof(float));
        if (!ok) return det_fail(SDB_FORMAT, "truncated checkpoint file");
    }
    uint64_t nvel = 0;
    pod(nvel);
    size_t total = 0;
    for (const auto& w : ws) total += w.size();
    // validate before allocating: a corrupt or hostile length must not throw
    // out of the C ABI (bad_alloc / length_error)
    if (!ok) return det_fail(SDB_FORMAT, "truncated checkpoint file");
    if (nvel != total) return det_fail(SDB_FORMAT, "checkpoint velocity length differs from the parameters");
    std::vector<float> vel(static_cast<size_t>(nvel));
    bytes(vel.data(), vel.size() * sizeof(float));
    double scale = 0.0, growth = 0.0, backoff = 0.0, mn = 0.0, mx = 0.0;
    int64_t good = 0, gi = 0;
    uint8_t mode = 0;
    uint32_t nrun = 0;
    pod(scale); pod(good); pod(mode); pod(gi); pod(growth); pod(backoff); pod(mn); pod(mx); pod(nrun);
    if (!ok) return det_fail(SDB_FORMAT, "truncated checkpoint file");
    // running-stat blocks are skipped (IABN keeps none; a BN checkpoint's stats are not step state here)
    for (uint32_t i = 0; i < nrun; ++i) {
        float mom = 0.f;
        uint64_t c = 0;
        pod(mom);
        pod(c);
        if (!ok || c > (uint64_t{1} << 32)) return det_fail(SDB_FORMAT, "truncated checkpoint file");
        f.seekg(static_cast<std::streamoff>(2 * c * sizeof(float)), std::ios::cur);
    }
    size_t off = 0;
    for (uint32_t i = 0; i < np; ++i) {
        if (int rc = param_xfer(d, static_cast<int>(i), ws[i].data(), 1)) return rc;
        if (int rc = param_xfer(d, static_cast<int>(i), vel.data() + off, 4)) return rc;
        off += ws[i].size();
    }
    try {
        CK(cudaMemcpyAsync(d->scale, &scale, 8, cudaMemcpyHostToDevice, d->ctx->stream));
        CK(cudaMemcpyAsync(d->good, &good, 8, cudaMemcpyHostToDevice, d->ctx->stream));
        CK(cudaStreamSynchronize(d->ctx->stream));
    } catch (const std::exception& e) {
        return det_fail(SDB_CUDA, e.what());
    }
    if (config_digest) *config_digest = digest;
    if (step) *step = st;
    return SDB_OK;
}

int sdb_det_load_checkpoint(sdb_det* d, const char* path, uint64_t* config_digest, int64_t* step) {
    try {
        return load_checkpoint_impl(d, path, config_digest, step);
    } catch (const std::bad_alloc&) {
        return det_fail(SDB_FORMAT, "checkpoint sizes exceed host memory");
    } catch (const std::exception& e) {
        return det_fail(SDB_FORMAT, std::string("checkpoint: ") + e.what());
    }
}

// next pinned staging slot: waits (host) only for the H2D copies that read it
// two calls ago -- those sit at the start of an earlier step, so the host runs
// ahead of the device instead of draining the stream every step
static int stage_slot(sdb_det* d) {
    const int k = d->stage_next;
    d->stage_next = (k + 1) % sdb_det::kStage;
    if (d->stage_busy[k]) CK(cudaEventSynchronize(d->stage_ev[k]));
    d->stage_busy[k] = false;
    return k;
}

static void stage_done(sdb_det* d, int k) {
    CK(cudaEventRecord(d->stage_ev[k], d->ctx->stream));
    d->stage_busy[k] = true;
}

static void stage_gt(sdb_det* d, const float* gt_boxes, const int32_t* gt_cls, const int32_t* gt_count,
                     const int64_t* slots) {
    const auto& cf = d->cfg;
    const int b = cf.batch;
    const int k = stage_slot(d);
    std::memcpy(d->h_gt[k], gt_boxes, static_cast<size_t>(b) * cf.max_gt * 16);
    std::memcpy(d->h_cls[k], gt_cls, static_cast<size_t>(b) * cf.max_gt * 4);
    for (int j = 0; j < b; ++j) d->h_cnt[k][j] = std::min(std::max(gt_count[j], 0), cf.max_gt);
    for (int j = 0; j < b; ++j) {
        d->h_keys[k][j] = mix64(cf.seed ^ 0xA11C0000ull, static_cast<uint64_t>(slots[j]));
        d->h_keys[k][b + j] = mix64(cf.seed ^ 0x5A3B0000ull, static_cast<uint64_t>(slots[j]));
    }
    cudaStream_t st = d->ctx->stream;
    CK(cudaMemcpyAsync(d->gt, d->h_gt[k], static_cast<size_t>(b) * cf.max_gt * 16, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d->gt_cls, d->h_cls[k], static_cast<size_t>(b) * cf.max_gt * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d->gt_count, d->h_cnt[k], b * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d->keys, d->h_keys[k], 2 * b * 8, cudaMemcpyHostToDevice, st));
    stage_done(d, k);
}

int sdb_det_set_batch(sdb_det* d, const void* images, int on_host, const float* gt_boxes, const int32_t* gt_cls,
                      const int32_t* gt_count, const int64_t* slots) {
    try {
        cudaStream_t st = d->ctx->stream;
        // stream-ordered behind the previous step; `images` must stay valid
        // until this batch's step has consumed it (as for any async copy)
        if (images)
            CK(cudaMemcpyAsync(d->img.p, images, d->img.numel() * d->es,
                               on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
        stage_gt(d, gt_boxes, gt_cls, gt_count, slots);
    } catch (const std::exception& e) {
        return det_fail(SDB_CUDA, e.what());
    }
    return SDB_OK;
}

int sdb_det_synth_images(sdb_det* d, const int64_t* slots) {
    try {
        // stream-ordered after the previous step (never touch the step workspace:
        // the previous step may still be running on the context stream)
        cudaStream_t st = d->ctx->stream;
        const int k = stage_slot(d);
        std::memcpy(d->h_slots[k], slots, d->cfg.batch * 8);
        CK(cudaMemcpyAsync(d->slots_dev, d->h_slots[k], d->cfg.batch * 8, cudaMemcpyHostToDevice, st));
        stage_done(d, k);
        CK(synth_images(d->dt, d->img.p, d->cfg.batch, d->cfg.img_h, d->cfg.img_w, 8, d->cfg.seed, d->slots_dev, 0, st));
    } catch (const std::exception& e) {
        return det_fail(SDB_CUDA, e.what());
    }
    return SDB_OK;
}

int sdb_det_step(sdb_det* d) {
    try {
        cudaStream_t st = d->ctx->stream;
        if (!d->use_graph || d->steps_done == 0) {
            run_step(d);
        } else {
            if (!d->gexec) {
                cudaGraph_t graph;
                CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
                run_step(d);
                CK(cudaStreamEndCapture(st, &graph));
                size_t n = 0;
                CK(cudaGraphGetNodes(graph, nullptr, &n));
                std::vector<cudaGraphNode_t> nodes(n);
                CK(cudaGraphGetNodes(graph, nodes.data(), &n));
                int64_t k = 0;
                for (auto nd : nodes) {
                    cudaGraphNodeType t;
                    CK(cudaGraphNodeGetType(nd, &t));
                    k += t == cudaGraphNodeTypeKernel;
                }
                d->launches = k;
                CK(cudaGraphInstantiate(&d->gexec, graph, 0));
                CK(cudaGraphDestroy(graph));
            }
            CK(cudaGraphLaunch(d->gexec, st));
        }
        ++d->steps_done;
    } catch (const CollectiveFailure& e) {
        return det_fail(SDB_COLLECTIVE, e.what());
    } catch (const std::exception& e) {
        return det_fail(SDB_CUDA, e.what());
    }
    return SDB_OK;
}

int sdb_det_read_losses(sdb_det* d, double* losses5, double* scale_used, int* overflow) {
    try {
        cudaStream_t st = d->ctx->stream;
        CK(cudaMemcpyAsync(d->h_losses, d->losses, 4 * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(d->h_losses + 8, d->scale_used, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(d->h_losses + 9, d->flag, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double K = d->ctx->world;
        double tot = 0;
        for (int i = 0; i < 4; ++i) {
            if (losses5) losses5[i] = d->h_losses[i] / K;
            tot += d->h_losses[i];
        }
        if (losses5) losses5[4] = tot / K;
        if (scale_used) *scale_used = d->h_losses[8];
        if (overflow) *overflow = *reinterpret_cast<int*>(d->h_losses + 9);
    } catch (const std::exception& e) {
        return det_fail(SDB_CUDA, e.what());
    }
    return SDB_OK;
}

int sdb_det_train_step_host(sdb_det* d, const void* images_host, const float* gt_boxes, const int32_t* gt_cls,
                            const int32_t* gt_count, const int64_t* slots, double* losses5) {
    try {
        cudaStream_t st = d->ctx->stream;
        CK(cudaMemcpyAsync(d->img.p, images_host, d->img.numel() * d->es, cudaMemcpyHostToDevice, st));
        stage_gt(d, gt_boxes, gt_cls, gt_count, slots);
    } catch (const std::exception& e) {
        return det_fail(SDB_CUDA, e.what());
    }
    if (int rc = sdb_det_step(d)) return rc;
    return sdb_det_read_losses(d, losses5, nullptr, nullptr);
}

int sdb_det_train_step_host_nchw(sdb_det* d, const void* images_nchw_host, const float* gt_boxes,
                                 const int32_t* gt_cls, const int32_t* gt_count, const int64_t* slots,
                                 double* losses5) {
    try {
        cudaStream_t st = d->ctx->stream;
        const size_t bytes = static_cast<size_t>(d->img.n) * 3 * d->img.h * d->img.w * d->es;
        if (!d->img3) d->img3 = d->alloc(bytes);
        // only the 3 real channels cross PCIe; the 8-channel padding happens on device
        CK(cudaMemcpyAsync(d->img3, images_nchw_host, bytes, cudaMemcpyHostToDevice, st));
        CK(nchw3_to_nhwc(d->dt, d->img3, d->img.n, d->img.h, d->img.w, d->img.c, d->img.p, st));
        stage_gt(d, gt_boxes, gt_cls, gt_count, slots);
    } catch (const std::exception& e) {
        return det_fail(SDB_CUDA, e.what());
    }
    if (int rc = sdb_det_step(d)) return rc;
    return sdb_det_read_losses(d, losses5, nullptr, nullptr);
}

int sdb_det_export(sdb_det* d, int what, void* host, int64_t cap, int64_t* bytes) {
    const auto& cf = d->cfg;
    const void* src = nullptr;
    int64_t n = 0;
    double tmp_state[2];
    switch (what) {
        case 0: src = d->a_labels; n = static_cast<int64_t>(cf.batch) * d->nA; break;
        case 1: src = d->a_targets; n = static_cast<int64_t>(cf.batch) * d->nA * 16; break;
        case 2: src = d->props; n = static_cast<int64_t>(cf.batch) * cf.post_nms * 16; break;
        case 3: src = d->prop_count; n = cf.batch * 4; break;
        case 4: src = d->rois; n = static_cast<int64_t>(d->R) * 20; break;
        case 5: src = d->roi_labels; n = static_cast<int64_t>(d->R) * 4; break;
        case 6: src = d->roi_targets; n = static_cast<int64_t>(d->R) * 16; break;
        case 7: src = d->rpn_logits.p; n = d->rpn_logits.numel() * d->es; break;
        case 8: src = d->rpn_deltas.p; n = d->rpn_deltas.numel() * d->es; break;
        case 9: src = d->anchors; n = static_cast<int64_t>(d->nA) * 16; break;
        case 10: src = d->c4.p; n = d->c4.numel() * d->es; break;
        case 11: src = d->img.p; n = d->img.numel() * d->es; break;
        case 13: src = d->stem_z.p; n = d->stem_z.numel() * d->es; break;
        case 14: src = d->pool.p; n = d->pool.numel() * d->es; break;
        case 15: src = d->stem_x2; n = d->stem_x2 ? static_cast<int64_t>(d->stem2.g.W) * 192 * 2 : 0; break;
        case 16: src = d->wdev; n = d->n_w * d->es; break;
        case 17: src = d->w32; n = d->n_w * 4; break;
        case 18: src = d->roi_feat.p; n = d->roi_feat.numel() * d->es; break;
        case 19:
            if (d->head_pool_fuse)
                return det_fail(SDB_PARAM, "head_out is pooled inside the last head block and not stored "
                                           "(build the detector with SDB_NO_HEAD_POOL_FUSE=1 to export it)");
            src = d->head_out.p; n = d->head_out.numel() * d->es; break;
        case 20: src = d->pooled.p; n = d->pooled.numel() * d->es; break;
        case 21: src = d->cls_logits.p; n = d->cls_logits.numel() * d->es; break;
        case 22: src = d->bbox_pred.p; n = d->bbox_pred.numel() * d->es; break;
        case 12: {
            cudaStreamSynchronize(d->ctx->stream);
            cudaMemcpy(&tmp_state[0], d->scale, 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(&tmp_state[1], d->good, 8, cudaMemcpyDeviceToHost);
            if (bytes) *bytes = 16;
            if (host && cap >= 16) std::memcpy(host, tmp_state, 16);
            return SDB_OK;
        }
        default: return det_fail(SDB_PARAM, "unknown export id");
    }
    if (bytes) *bytes = n;
    if (!host) return SDB_OK;
    if (cap < n) return det_fail(SDB_PARAM, "export buffer too small");
    if (cudaStreamSynchronize(d->ctx->stream) != cudaSuccess || cudaMemcpy(host, src, n, cudaMemcpyDeviceToHost) != cudaSuccess)
        return det_fail(SDB_CUDA, "export copy failed");
    return SDB_OK;
}

int sdb_det_dims(sdb_det* d, int* fh, int* fw, int* A, int* A_pad) {
    if (fh) *fh = d->fh;
    if (fw) *fw = d->fw;
    if (A) *A = d->A;
    if (A_pad) *A_pad = d->A_pad;
    return SDB_OK;
}

int sdb_det_profile(sdb_det* d, double* ms, double* flops, double* bytes, int64_t* launches, int ncat) {
    try {
        Prof& p = d->prof;
        p.used = 0;
        p.recs.clear();
        p.labels.clear();
        p.rec_flops.clear();
        p.rec_bytes.clear();
        std::fill(p.flops, p.flops + P_NCAT, 0.0);
        std::fill(p.bytes, p.bytes + P_NCAT, 0.0);
        std::fill(p.launches, p.launches + P_NCAT, 0);
        p.on = true;
        run_step(d);
        p.on = false;
        CK(cudaStreamSynchronize(d->ctx->stream));
        std::vector<double> acc(P_NCAT, 0.0);
        const bool verbose = std::getenv("SDB_PROFILE_VERBOSE") != nullptr;
        p.last.clear();
        for (size_t k = 0; k < p.recs.size(); ++k) {
            auto& r = p.recs[k];
            float t = 0;
            CK(cudaEventElapsedTime(&t, r.second.first, r.second.second));
            acc[r.first] += t;
            if (!p.labels[k].empty()) p.last.push_back({r.first, p.labels[k], t, p.rec_flops[k], p.rec_bytes[k]});
            if (verbose && !p.labels[k].empty())
                std::fprintf(stderr, "[sdb-prof] %-60s %8.1f us %7.0f TF/s %7.0f GB/s\n", p.labels[k].c_str(),
                             t * 1e3, p.rec_flops[k] / (t * 1e-3) / 1e12, p.rec_bytes[k] / (t * 1e-3) / 1e9);
        }
        p.labels.clear();
        p.rec_flops.clear();
        p.rec_bytes.clear();
        for (int i = 0; i < ncat && i < P_NCAT; ++i) {
            if (ms) ms[i] = acc[i];
            if (flops) flops[i] = p.flops[i];
            if (bytes) bytes[i] = p.bytes[i];
            if (launches) launches[i] = p.launches[i];
        }
        ++d->steps_done;
    } catch (const std::exception& e) {
        d->prof.on = false;
        return det_fail(SDB_CUDA, e.what());
    }
    return SDB_OK;
}

int sdb_det_profile_record(sdb_det* d, int k, int* cat, char* label, int cap, double* ms, double* flops,
                           double* bytes) {
    if (!d) return det_fail(SDB_CONTRACT, "null detector");
    const auto& L = d->prof.last;
    if (k < 0) return static_cast<int>(L.size());
    if (k >= static_cast<int>(L.size())) return det_fail(SDB_PARAM, "profile record index out of range");
    const auto& r = L[static_cast<size_t>(k)];
    if (cat) *cat = r.cat;
    if (label && cap > 0) {
        std::strncpy(label, r.label.c_str(), static_cast<size_t>(cap) - 1);
        label[cap - 1] = 0;
    }
    if (ms) *ms = r.ms;
    if (flops) *flops = r.flops;
    if (bytes) *bytes = r.bytes;
    return SDB_OK;
}

int sdb_det_kernel_launches(sdb_det* d, int64_t* n) {
    *n = d->launches;
    return SDB_OK;
}

int sdb_plan_checkpoints(int L, int* starts, int cap) {
    if (L < 1) return det_fail(SDB_PARAM, "layer count must be >= 1");
    const std::vector<int> st = plan_segments(L);
    if (static_cast<int>(st.size()) > cap) return det_fail(SDB_PARAM, "starts capacity too small");
    std::copy(st.begin(), st.end(), starts);
    return static_cast<int>(st.size()) - 1;
}

int sdb_det_memory(sdb_det* d, int64_t* backbone_act_bytes, int64_t* device_bytes, int* segments) {
    if (!d) return det_fail(SDB_CONTRACT, "null detector");
    if (backbone_act_bytes) *backbone_act_bytes = d->bytes_backbone;
    if (device_bytes) *device_bytes = d->bytes_total;
    if (segments) *segments = d->ck_start.empty() ? 0 : static_cast<int>(d->ck_start.size()) - 1;
    return SDB_OK;
}

}  // extern "C"
