// oracle/detector_ref.cpp -- TEST INFRASTRUCTURE ONLY.
//
// The Faster R-CNN C4 training step restated ON THE REFERENCE ENGINE: the
// forward/backward runs on simdet::Tape (src/autograd.cpp) with the
// reference's own conv2d, matmul, add, relu, leaky_relu, reduce_mean, and the
// reference BN / IABN math (syncbn_forward/backward, iabn_forward/backward)
// wrapped in CustomOps exactly like make_bn_op / make_iabn_op
// (src/model.cpp:17-96, which live in an anonymous namespace there).  The
// operators the reference lacks (max-pool, RoIAlign, RPN BCE, smooth-L1, the
// CE op of model.cpp:101-151) are plugged in as CustomOps over the restated
// kernels of oracle/restate.cpp, following the same fp16 contract: every op
// output is a Tensor of the input dtype (rounded RNE on construction,
// src/tensor.cpp:59-82), gradients are finalised in the node's dtype by the
// tape (src/autograd.cpp:437-440,475-485).
//
// Discrete decisions (anchor labels, sampled RoIs) are INPUTS here ("teacher
// forcing"): the parity tests check them separately and bit-exactly with the
// restated proposal/target code, then feed the GPU's decisions so the
// continuous part of the step is compared on identical samples.
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "restate.hpp"
#include "simdet/autograd.hpp"
#include "simdet/memopt.hpp"
#include "simdet/precision.hpp"
#include "simdet/syncbn.hpp"
#include "simdet/tensor.hpp"

using namespace simdet;

extern "C" {
struct RefDetCfg {
    int mode, batch, img_h, img_w;
    int blocks[4];
    int num_classes, rpn_channels, A, pool, sampling_ratio, rpn_batch;
    float eps, slope;
};
}

namespace {

Tensor vec_tensor(const std::vector<float>& v) { return Tensor({static_cast<int64_t>(v.size())}, DType::F32, v); }

// make_bn_op (src/model.cpp:17-45), group == nullptr
std::shared_ptr<CustomOp> bn_op(float eps) {
    auto op = std::make_shared<CustomOp>();
    op->name = "bn";
    op->saved_inputs = {0, 1};
    op->forward = [eps](const std::vector<const Tensor*>& in, std::vector<Tensor>& stash) {
        auto [y, st] = syncbn_forward(*in[0], in[1]->data(), in[2]->data(), eps, nullptr);
        stash.push_back(vec_tensor(st.mean));
        stash.push_back(vec_tensor(st.invstd));
        stash.push_back(Tensor::scalar(static_cast<float>(st.count)));
        return std::move(y);
    };
    op->backward = [](const Tensor& dy, const std::vector<const Tensor*>& in, const Tensor*,
                      const std::vector<Tensor>& stash) {
        BNStats st;
        st.mean.assign(stash[0].data().begin(), stash[0].data().end());
        st.invstd.assign(stash[1].data().begin(), stash[1].data().end());
        st.count = static_cast<int64_t>(stash[2][0]);
        BnGrads g = syncbn_backward(dy, *in[0], st, in[1]->data(), nullptr);
        std::vector<Tensor> out;
        out.push_back(std::move(g.dx));
        out.push_back(vec_tensor(g.dgamma));
        out.push_back(vec_tensor(g.dbeta));
        return out;
    };
    return op;
}

// make_iabn_op (src/model.cpp:49-96)
std::shared_ptr<CustomOp> iabn_op(float eps, float slope) {
    auto op = std::make_shared<CustomOp>();
    op->name = "iabn";
    op->saved_inputs = {1, 2};
    op->save_output = true;
    op->forward = [eps, slope](const std::vector<const Tensor*>& in, std::vector<Tensor>& stash) {
        auto [y, sv] = iabn_forward(*in[0], in[1]->data(), in[2]->data(), eps, slope);
        stash.push_back(vec_tensor(sv.mean));
        stash.push_back(vec_tensor(sv.invstd));
        return std::move(y);
    };
    op->backward = [eps, slope](const Tensor& dy, const std::vector<const Tensor*>& in, const Tensor* out,
                                const std::vector<Tensor>& stash) {
        IabnSaved sv;
        sv.y = *out;
        sv.mean.assign(stash[0].data().begin(), stash[0].data().end());
        sv.invstd.assign(stash[1].data().begin(), stash[1].data().end());
        sv.gamma.assign(in[1]->data().begin(), in[1]->data().end());
        sv.beta.assign(in[2]->data().begin(), in[2]->data().end());
        sv.eps = eps;
        sv.slope = slope;
        IabnGrads g = iabn_backward(dy, sv);
        std::vector<Tensor> res;
        res.push_back(std::move(g.dx));
        res.push_back(vec_tensor(g.dgamma));
        res.push_back(vec_tensor(g.dbeta));
        return res;
    };
    return op;
}

std::shared_ptr<CustomOp> maxpool_op() {
    auto op = std::make_shared<CustomOp>();
    op->name = "maxpool";
    op->saved_inputs = {0};
    op->forward = [](const std::vector<const Tensor*>& in, std::vector<Tensor>&) {
        const Shape& s = in[0]->shape();
        const int N = s[0], C = s[1], H = s[2], W = s[3];
        const int Ho = (H + 2 - 3) / 2 + 1, Wo = (W + 2 - 3) / 2 + 1;
        std::vector<float> y(static_cast<size_t>(N) * C * Ho * Wo);
        orc_maxpool_fwd(in[0]->data().data(), N, C, H, W, 3, 2, 1, y.data());
        return Tensor({N, C, Ho, Wo}, in[0]->dtype(), std::move(y));
    };
    op->backward = [](const Tensor& dy, const std::vector<const Tensor*>& in, const Tensor*,
                      const std::vector<Tensor>&) {
        const Shape& s = in[0]->shape();
        std::vector<float> dx(static_cast<size_t>(in[0]->numel()));
        orc_maxpool_bwd(in[0]->data().data(), dy.data().data(), s[0], s[1], s[2], s[3], 3, 2, 1, dx.data());
        std::vector<Tensor> r;
        r.push_back(Tensor(s, DType::F32, std::move(dx)));
        return r;
    };
    return op;
}

std::shared_ptr<CustomOp> roialign_op(std::vector<float> rois, int P, int sr, Shape feat_shape) {
    auto op = std::make_shared<CustomOp>();
    op->name = "roialign";
    auto rp = std::make_shared<std::vector<float>>(std::move(rois));
    op->forward = [rp, P, sr](const std::vector<const Tensor*>& in, std::vector<Tensor>&) {
        const Shape& s = in[0]->shape();
        const int64_t R = static_cast<int64_t>(rp->size() / 5);
        std::vector<float> y(static_cast<size_t>(R) * s[1] * P * P);
        orc_roialign_fwd(in[0]->data().data(), s[0], s[1], s[2], s[3], rp->data(), R, P, 1.0f / 16.0f, sr, 1,
                         y.data());
        return Tensor({R, s[1], P, P}, in[0]->dtype(), std::move(y));
    };
    op->backward = [rp, P, sr, feat_shape](const Tensor& dy, const std::vector<const Tensor*>&, const Tensor*,
                                           const std::vector<Tensor>&) {
        const Shape& s = feat_shape;
        const int64_t R = static_cast<int64_t>(rp->size() / 5);
        std::vector<float> dx(static_cast<size_t>(s[0] * s[1] * s[2] * s[3]));
        orc_roialign_bwd(dy.data().data(), s[0], s[1], s[2], s[3], rp->data(), R, P, 1.0f / 16.0f, sr, 1, dx.data());
        std::vector<Tensor> r;
        r.push_back(Tensor(s, DType::F32, std::move(dx)));
        return r;
    };
    return op;
}

// RPN sigmoid BCE over anchors, logits NCHW [N, A, H, W]; anchor a_idx = (h*W+w)*A + a
std::shared_ptr<CustomOp> rpn_bce_op(std::vector<int8_t> labels, int A, double grad_scale, double* loss_out) {
    auto op = std::make_shared<CustomOp>();
    op->name = "rpn_bce";
    op->output_tag = "loss";
    op->saved_inputs = {0};
    auto lab = std::make_shared<std::vector<int8_t>>(std::move(labels));
    auto gather = [lab, A](const Tensor& x, std::vector<float>& flat) {
        const Shape& s = x.shape();
        const int64_t N = s[0], H = s[2], W = s[3];
        flat.resize(static_cast<size_t>(N * H * W * A));
        for (int64_t n = 0; n < N; ++n)
            for (int64_t a = 0; a < A; ++a)
                for (int64_t h = 0; h < H; ++h)
                    for (int64_t w = 0; w < W; ++w)
                        flat[((n * H + h) * W + w) * A + a] = x[((n * s[1] + a) * H + h) * W + w];
    };
    op->forward = [lab, gather, loss_out](const std::vector<const Tensor*>& in, std::vector<Tensor>&) {
        std::vector<float> flat;
        gather(*in[0], flat);
        int64_t cnt = 0;
        for (int8_t v : *lab) cnt += v >= 0;
        const double l = orc_sigmoid_bce(flat.data(), lab->data(), static_cast<int64_t>(flat.size()),
                                         static_cast<double>(cnt), 1.0, nullptr);
        if (loss_out) *loss_out = l;
        return Tensor::scalar(static_cast<float>(l));
    };
    op->backward = [lab, gather, A, grad_scale](const Tensor& dy, const std::vector<const Tensor*>& in, const Tensor*,
                                                const std::vector<Tensor>&) {
        std::vector<float> flat, g;
        gather(*in[0], flat);
        g.resize(flat.size());
        int64_t cnt = 0;
        for (int8_t v : *lab) cnt += v >= 0;
        orc_sigmoid_bce(flat.data(), lab->data(), static_cast<int64_t>(flat.size()), static_cast<double>(cnt),
                        static_cast<double>(dy[0]) * grad_scale, g.data());
        const Shape& s = in[0]->shape();
        const int64_t N = s[0], H = s[2], W = s[3];
        Tensor dx(s, DType::F32, 0.0f);
        for (int64_t n = 0; n < N; ++n)
            for (int64_t a = 0; a < A; ++a)
                for (int64_t h = 0; h < H; ++h)
                    for (int64_t w = 0; w < W; ++w)
                        dx[((n * s[1] + a) * H + h) * W + w] = g[((n * H + h) * W + w) * A + a];
        std::vector<Tensor> r;
        r.push_back(std::move(dx));
        return r;
    };
    return op;
}

// RPN smooth-L1 (beta 1/9) on deltas NCHW [N, 4A, H, W] for fg anchors
std::shared_ptr<CustomOp> rpn_sl1_op(std::vector<int8_t> labels, std::vector<float> targets, int A, double norm,
                                     double grad_scale, double* loss_out) {
    auto op = std::make_shared<CustomOp>();
    op->name = "rpn_sl1";
    op->output_tag = "loss";
    op->saved_inputs = {0};
    auto lab = std::make_shared<std::vector<int8_t>>(std::move(labels));
    auto tg = std::make_shared<std::vector<float>>(std::move(targets));
    auto gather = [A](const Tensor& x, std::vector<float>& flat) {
        const Shape& s = x.shape();
        const int64_t N = s[0], H = s[2], W = s[3];
        flat.resize(static_cast<size_t>(N * H * W * A * 4));
        for (int64_t n = 0; n < N; ++n)
            for (int64_t c = 0; c < 4 * A; ++c)
                for (int64_t h = 0; h < H; ++h)
                    for (int64_t w = 0; w < W; ++w)
                        flat[((n * H + h) * W + w) * 4 * A + c] = x[((n * s[1] + c) * H + h) * W + w];
    };
    op->forward = [lab, tg, gather, norm, loss_out](const std::vector<const Tensor*>& in, std::vector<Tensor>&) {
        std::vector<float> flat;
        gather(*in[0], flat);
        std::vector<float> wgt(lab->size());
        for (size_t i = 0; i < lab->size(); ++i) wgt[i] = (*lab)[i] == 1 ? 1.0f : 0.0f;
        const double l = orc_smooth_l1(flat.data(), tg->data(), wgt.data(), static_cast<int64_t>(lab->size()),
                                       1.0 / 9.0, norm, 1.0, nullptr);
        if (loss_out) *loss_out = l;
        return Tensor::scalar(static_cast<float>(l));
    };
    op->backward = [lab, tg, gather, A, norm, grad_scale](const Tensor& dy, const std::vector<const Tensor*>& in,
                                                          const Tensor*, const std::vector<Tensor>&) {
        std::vector<float> flat, g;
        gather(*in[0], flat);
        g.resize(flat.size());
        std::vector<float> wgt(lab->size());
        for (size_t i = 0; i < lab->size(); ++i) wgt[i] = (*lab)[i] == 1 ? 1.0f : 0.0f;
        orc_smooth_l1(flat.data(), tg->data(), wgt.data(), static_cast<int64_t>(lab->size()), 1.0 / 9.0, norm,
                      static_cast<double>(dy[0]) * grad_scale, g.data());
        const Shape& s = in[0]->shape();
        const int64_t N = s[0], H = s[2], W = s[3];
        Tensor dx(s, DType::F32, 0.0f);
        for (int64_t n = 0; n < N; ++n)
            for (int64_t c = 0; c < 4 * A; ++c)
                for (int64_t h = 0; h < H; ++h)
                    for (int64_t w = 0; w < W; ++w)
                        dx[((n * s[1] + c) * H + h) * W + w] = g[((n * H + h) * W + w) * 4 * A + c];
        std::vector<Tensor> r;
        r.push_back(std::move(dx));
        return r;
    };
    return op;
}

// the reference CE op (src/model.cpp:101-151), restated because it is file-local there
std::shared_ptr<CustomOp> ce_op(std::vector<int32_t> labels, double grad_scale, double* loss_out) {
    auto op = std::make_shared<CustomOp>();
    op->name = "softmax_ce";
    op->output_tag = "loss";
    op->saved_inputs = {0};
    auto lab = std::make_shared<std::vector<int32_t>>(std::move(labels));
    op->forward = [lab, loss_out](const std::vector<const Tensor*>& in, std::vector<Tensor>&) {
        const Shape& s = in[0]->shape();
        const double l = orc_softmax_ce(in[0]->data().data(), s[0], s[1], lab->data(), 1.0, 1.0, nullptr);
        if (loss_out) *loss_out = l;
        return Tensor::scalar(static_cast<float>(l));
    };
    op->backward = [lab, grad_scale](const Tensor& dy, const std::vector<const Tensor*>& in, const Tensor*,
                                     const std::vector<Tensor>&) {
        const Shape& s = in[0]->shape();
        Tensor dx(s, DType::F32, 0.0f);
        orc_softmax_ce(in[0]->data().data(), s[0], s[1], lab->data(), static_cast<double>(dy[0]), grad_scale,
                       dx.data().data());
        std::vector<Tensor> r;
        r.push_back(std::move(dx));
        return r;
    };
    return op;
}

// class-specific smooth-L1 (beta 1) on pred [R, 4*ncls] at the label's slot, normalised by R
std::shared_ptr<CustomOp> rcnn_sl1_op(std::vector<int32_t> labels, std::vector<float> targets, double grad_scale,
                                      double* loss_out) {
    auto op = std::make_shared<CustomOp>();
    op->name = "rcnn_sl1";
    op->output_tag = "loss";
    op->saved_inputs = {0};
    auto lab = std::make_shared<std::vector<int32_t>>(std::move(labels));
    auto tg = std::make_shared<std::vector<float>>(std::move(targets));
    auto pick = [lab](const Tensor& x, std::vector<float>& sel, std::vector<float>& wgt) {
        const int64_t R = x.shape()[0], ld = x.shape()[1];
        sel.assign(static_cast<size_t>(R * 4), 0.0f);
        wgt.assign(static_cast<size_t>(R), 0.0f);
        for (int64_t r = 0; r < R; ++r) {
            const int l = (*lab)[r];
            if (l <= 0) continue;
            wgt[r] = 1.0f;
            for (int k = 0; k < 4; ++k) sel[r * 4 + k] = x[r * ld + 4 * l + k];
        }
    };
    op->forward = [lab, tg, pick, loss_out](const std::vector<const Tensor*>& in, std::vector<Tensor>&) {
        std::vector<float> sel, wgt;
        pick(*in[0], sel, wgt);
        const int64_t R = in[0]->shape()[0];
        const double l = orc_smooth_l1(sel.data(), tg->data(), wgt.data(), R, 1.0, static_cast<double>(R), 1.0, nullptr);
        if (loss_out) *loss_out = l;
        return Tensor::scalar(static_cast<float>(l));
    };
    op->backward = [lab, tg, pick, grad_scale](const Tensor& dy, const std::vector<const Tensor*>& in, const Tensor*,
                                               const std::vector<Tensor>&) {
        std::vector<float> sel, wgt;
        pick(*in[0], sel, wgt);
        const int64_t R = in[0]->shape()[0], ld = in[0]->shape()[1];
        std::vector<float> g(sel.size());
        orc_smooth_l1(sel.data(), tg->data(), wgt.data(), R, 1.0, static_cast<double>(R),
                      static_cast<double>(dy[0]) * grad_scale, g.data());
        Tensor dx(in[0]->shape(), DType::F32, 0.0f);
        for (int64_t r = 0; r < R; ++r) {
            const int l = (*lab)[r];
            if (l <= 0) continue;
            for (int k = 0; k < 4; ++k) dx[r * ld + 4 * l + k] = g[r * 4 + k];
        }
        std::vector<Tensor> res;
        res.push_back(std::move(dx));
        return res;
    };
    return op;
}

struct PSpec {
    std::string name;
    Shape shape;
    int kind;  // 0 conv, 1 fc, 2 gamma, 3 beta
};

struct Net {
    const RefDetCfg& c;
    std::vector<PSpec> specs;
    explicit Net(const RefDetCfg& cfg) : c(cfg) {}
    void conv(const std::string& n, int cin, int cout, int k) { specs.push_back({n, {cout, cin, k, k}, 0}); }
    void norm(const std::string& n, int C) {
        specs.push_back({n + ".gamma", {C}, 2});
        specs.push_back({n + ".beta", {C}, 3});
    }
    void stage(const std::string& pref, int nb, int cin, int width, int cout) {
        for (int b = 0; b < nb; ++b) {
            const std::string p = pref + "." + std::to_string(b);
            const int ci = b == 0 ? cin : cout;
            conv(p + ".conv1", ci, width, 1);
            norm(p + ".bn1", width);
            conv(p + ".conv2", width, width, 3);
            norm(p + ".bn2", width);
            conv(p + ".conv3", width, cout, 1);
            norm(p + ".bn3", cout);
            if (b == 0) {
                conv(p + ".down", ci, cout, 1);
                norm(p + ".down_bn", cout);
            }
        }
    }
    void build() {
        conv("stem.conv", 3, 64, 7);
        norm("stem.bn", 64);
        stage("res2", c.blocks[0], 64, 64, 256);
        stage("res3", c.blocks[1], 256, 128, 512);
        stage("res4", c.blocks[2], 512, 256, 1024);
        conv("rpn.conv", 1024, c.rpn_channels, 3);
        specs.push_back({"rpn.cls", {c.A, c.rpn_channels, 1, 1}, 0});
        specs.push_back({"rpn.bbox", {4 * c.A, c.rpn_channels, 1, 1}, 0});
        int feat = 1024;
        if (c.blocks[3] > 0) {
            stage("res5", c.blocks[3], 1024, 512, 2048);
            feat = 2048;
        }
        specs.push_back({"fc.cls", {feat, c.num_classes + 1}, 1});
        specs.push_back({"fc.bbox", {feat, 4 * (c.num_classes + 1)}, 1});
    }
};

int64_t numel(const Shape& s) {
    int64_t n = 1;
    for (int64_t d : s) n *= d;
    return n;
}

}  // namespace

extern "C" {

// parameter list in pack order: writes up to `cap` names (64 chars each) and
// shapes (4 int64 each); returns the count
int ref_det_param_list(const RefDetCfg* cfg, char* names, int64_t* shapes, int* kinds, int cap) {
    Net net(*cfg);
    net.build();
    const int n = static_cast<int>(net.specs.size());
    for (int i = 0; i < n && i < cap; ++i) {
        if (names) {
            std::strncpy(names + 64 * i, net.specs[i].name.c_str(), 63);
            names[64 * i + 63] = 0;
        }
        if (shapes)
            for (int k = 0; k < 4; ++k)
                shapes[4 * i + k] = k < static_cast<int>(net.specs[i].shape.size()) ? net.specs[i].shape[k] : 1;
        if (kinds) kinds[i] = net.specs[i].kind;
    }
    return n;
}

// One training step's forward + backward on the reference Tape with the given
// (teacher-forced) targets.  params/grads: concatenated reference layouts in
// pack order (fp32 masters; conv/fc cast to fp16 shadows in mode 1, src/trainer.cpp:222-227).
int ref_det_step(const RefDetCfg* cfg, const float* params, const float* images, const int8_t* a_labels,
                 const float* a_targets, const float* rois, const int32_t* roi_labels, const float* roi_targets, int R,
                 double grad_scale, double* losses4, float* grads, float* rpn_logits_out, float* rpn_deltas_out) {
    try {
        const RefDetCfg& c = *cfg;
        const DType dt = c.mode == 1 ? DType::F16 : DType::F32;
        Net net(c);
        net.build();
        Tape t;
        std::vector<ValueId> pid(net.specs.size());
        const float* pp = params;
        for (size_t i = 0; i < net.specs.size(); ++i) {
            const auto& s = net.specs[i];
            const int64_t n = numel(s.shape);
            Tensor v(s.shape, DType::F32, std::vector<float>(pp, pp + n));
            if (s.kind <= 1 && c.mode == 1) v = to_half(v);
            pid[i] = t.leaf(std::move(v), true, false, "param");
            pp += n;
        }
        size_t pi = 0;
        auto next = [&]() { return pid[pi++]; };
        const int N = c.batch;
        ValueId x = t.leaf(Tensor({N, 3, c.img_h, c.img_w}, dt,
                                  std::vector<float>(images, images + static_cast<int64_t>(N) * 3 * c.img_h * c.img_w)),
                           false);
        auto norm_act = [&](ValueId v, bool act, bool identity_iabn) {
            ValueId g = next(), b = next();
            if (c.mode == 0) {
                ValueId y = t.custom(bn_op(c.eps), {v, g, b});
                return act ? t.relu(y) : y;
            }
            return t.custom(iabn_op(c.eps, identity_iabn ? 1.0f : c.slope), {v, g, b});
        };
        auto block = [&](ValueId in, bool first, int stride) {
            ValueId w1 = next();
            ValueId h = t.conv2d(in, w1, first ? stride : 1, 0);
            h = norm_act(h, true, false);
            ValueId w2 = next();
            h = t.conv2d(h, w2, 1, 1);
            h = norm_act(h, true, false);
            ValueId w3 = next();
            h = t.conv2d(h, w3, 1, 0);
            h = norm_act(h, false, true);
            ValueId sc = in;
            if (first) {
                ValueId wd = next();
                sc = t.conv2d(in, wd, stride, 0);
                sc = norm_act(sc, false, true);
            }
            ValueId s = t.add(h, sc);
            return c.mode == 0 ? t.relu(s) : t.leaky_relu(s, c.slope);
        };
        auto stage = [&](ValueId in, int nb, int stride) {
            for (int b = 0; b < nb; ++b) in = block(in, b == 0, stride);
            return in;
        };
        // backbone
        ValueId h = t.conv2d(x, next(), 2, 3);
        h = norm_act(h, true, false);
        h = t.custom(maxpool_op(), {h});
        h = stage(h, c.blocks[0], 1);
        h = stage(h, c.blocks[1], 2);
        ValueId c4 = stage(h, c.blocks[2], 2);
        // RPN
        ValueId r = t.relu(t.conv2d(c4, next(), 1, 1));
        ValueId logits = t.conv2d(r, next(), 1, 0);
        ValueId deltas = t.conv2d(r, next(), 1, 0);
        if (rpn_logits_out) {
            const Tensor& lt = t.value(logits);
            std::memcpy(rpn_logits_out, lt.data().data(), lt.numel() * 4);
        }
        if (rpn_deltas_out) {
            const Tensor& dtn = t.value(deltas);
            std::memcpy(rpn_deltas_out, dtn.data().data(), dtn.numel() * 4);
        }
        const Shape c4s = t.value(c4).shape();
        const int64_t nA = c4s[2] * c4s[3] * c.A;
        std::vector<int8_t> al(a_labels, a_labels + N * nA);
        std::vector<float> atg(a_targets, a_targets + N * nA * 4);
        double l[4] = {0, 0, 0, 0};
        ValueId L1 = t.custom(rpn_bce_op(al, c.A, grad_scale, &l[0]), {logits});
        ValueId L2 = t.custom(rpn_sl1_op(al, atg, c.A, static_cast<double>(c.rpn_batch) * N, grad_scale, &l[1]),
                              {deltas});
        // RoI head
        std::vector<float> rv(rois, rois + static_cast<int64_t>(R) * 5);
        ValueId f = t.custom(roialign_op(rv, c.pool, c.sampling_ratio, c4s), {c4});
        if (c.blocks[3] > 0) f = stage(f, c.blocks[3], 2);
        ValueId pooled = t.reduce_mean(f, {2, 3});
        ValueId cls = t.matmul(pooled, next());
        ValueId box = t.matmul(pooled, next());
        std::vector<int32_t> rl(roi_labels, roi_labels + R);
        std::vector<float> rt(roi_targets, roi_targets + static_cast<int64_t>(R) * 4);
        ValueId L3 = t.custom(ce_op(rl, grad_scale, &l[2]), {cls});
        ValueId L4 = t.custom(rcnn_sl1_op(rl, rt, grad_scale, &l[3]), {box});
        ValueId total = t.add(t.add(t.add(L1, L2), L3), L4);
        GradMap g = t.backward(total);
        for (int i = 0; i < 4; ++i) losses4[i] = l[i];
        float* gp = grads;
        for (size_t i = 0; i < net.specs.size(); ++i) {
            const Tensor& gv = g.at(pid[i]);
            std::memcpy(gp, gv.data().data(), gv.numel() * 4);
            gp += gv.numel();
        }
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_det_step: %s\n", e.what());
        return 1;
    }
}

}  // extern "C"
