// oracle/restate.cpp -- TEST INFRASTRUCTURE ONLY (see restate.hpp header).
// CPU restatement of the SimpleDet C4 step operators; compiled with
// -O2 -ffp-contract=off so float/double expressions evaluate exactly as written.
#include "restate.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <utility>
#include <vector>

namespace {

struct BoxD {
    double x1, y1, x2, y2;
};

inline BoxD widen(const float* b) { return {b[0], b[1], b[2], b[3]}; }

// src/postproc.cpp:20-26 (area() from postproc.hpp:20)
inline double iou_d(const BoxD& a, const BoxD& b) {
    const double ix = std::max(0.0, std::min(a.x2, b.x2) - std::max(a.x1, b.x1));
    const double iy = std::max(0.0, std::min(a.y2, b.y2) - std::max(a.y1, b.y1));
    const double inter = ix * iy;
    const double area_a = (a.x2 - a.x1) * (a.y2 - a.y1);
    const double area_b = (b.x2 - b.x1) * (b.y2 - b.y1);
    const double uni = area_a + area_b - inter;
    return uni > 0.0 ? inter / uni : 0.0;
}

// (priority, index) ascending selection of the k smallest
std::vector<int64_t> pick_smallest(const std::vector<int64_t>& cand, uint64_t key, int64_t k) {
    std::vector<std::pair<uint64_t, int64_t>> pr;
    pr.reserve(cand.size());
    for (int64_t c : cand) pr.emplace_back(orc_mix64(key, static_cast<uint64_t>(c)), c);
    std::sort(pr.begin(), pr.end());
    std::vector<int64_t> out;
    for (int64_t i = 0; i < k && i < static_cast<int64_t>(pr.size()); ++i) out.push_back(pr[i].second);
    std::sort(out.begin(), out.end());
    return out;
}

inline float bilinear(const float* f, int H, int W, float y, float x) {
    if (y < -1.0f || y > static_cast<float>(H) || x < -1.0f || x > static_cast<float>(W)) return 0.0f;
    if (y <= 0.0f) y = 0.0f;
    if (x <= 0.0f) x = 0.0f;
    int yl = static_cast<int>(y), xl = static_cast<int>(x), yh, xh;
    if (yl >= H - 1) { yh = yl = H - 1; y = static_cast<float>(yl); } else yh = yl + 1;
    if (xl >= W - 1) { xh = xl = W - 1; x = static_cast<float>(xl); } else xh = xl + 1;
    const float ly = y - static_cast<float>(yl), lx = x - static_cast<float>(xl);
    const float hy = 1.0f - ly, hx = 1.0f - lx;
    const float w1 = hy * hx, w2 = hy * lx, w3 = ly * hx, w4 = ly * lx;
    return w1 * f[yl * W + xl] + w2 * f[yl * W + xh] + w3 * f[yh * W + xl] + w4 * f[yh * W + xh];
}

struct Corner {
    int yl, xl, yh, xh;
    float w1, w2, w3, w4;
    bool valid;
};

inline Corner corners(int H, int W, float y, float x) {
    Corner c{};
    if (y < -1.0f || y > static_cast<float>(H) || x < -1.0f || x > static_cast<float>(W)) {
        c.valid = false;
        return c;
    }
    c.valid = true;
    if (y <= 0.0f) y = 0.0f;
    if (x <= 0.0f) x = 0.0f;
    c.yl = static_cast<int>(y);
    c.xl = static_cast<int>(x);
    if (c.yl >= H - 1) { c.yh = c.yl = H - 1; y = static_cast<float>(c.yl); } else c.yh = c.yl + 1;
    if (c.xl >= W - 1) { c.xh = c.xl = W - 1; x = static_cast<float>(c.xl); } else c.xh = c.xl + 1;
    const float ly = y - static_cast<float>(c.yl), lx = x - static_cast<float>(c.xl);
    const float hy = 1.0f - ly, hx = 1.0f - lx;
    c.w1 = hy * hx; c.w2 = hy * lx; c.w3 = ly * hx; c.w4 = ly * lx;
    return c;
}

struct RoiGeom {
    int b;
    float sw, sh, bw, bh;
};

inline RoiGeom roi_geom(const float* r, int P, float scale, int aligned) {
    const float off = aligned ? 0.5f : 0.0f;
    RoiGeom g;
    g.b = static_cast<int>(r[0]);
    g.sw = r[1] * scale - off;
    g.sh = r[2] * scale - off;
    const float ew = r[3] * scale - off, eh = r[4] * scale - off;
    float rw = ew - g.sw, rh = eh - g.sh;
    if (!aligned) { rw = std::max(rw, 1.0f); rh = std::max(rh, 1.0f); }
    g.bw = rw / static_cast<float>(P);
    g.bh = rh / static_cast<float>(P);
    return g;
}

}  // namespace

extern "C" {

float orc_half_round(float f) {
    // independent of the reference's bit-twiddling: the compiler's IEEE
    // binary16 conversion (round-to-nearest-even, overflow to inf).
    return static_cast<float>(static_cast<_Float16>(f));
}

void orc_half_round_n(const float* in, float* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_half_round(in[i]);
}

float orc_expf(float xf) {
    // Range-reduced degree-11 Taylor in double with explicit +,* only, so the
    // CUDA path (__dmul_rn/__dadd_rn) evaluates the identical expression.
    const double x = xf;
    if (!(x == x)) return xf;
    if (x > 88.8) return std::numeric_limits<float>::infinity();
    if (x < -104.0) return 0.0f;
    const double kd = std::floor(x * 1.4426950408889634 + 0.5);
    const double r = (x - kd * 0.693147180369123816490) - kd * 1.90821492927058770002e-10;
    double p = 1.0 / 39916800.0;
    p = p * r + 1.0 / 3628800.0;
    p = p * r + 1.0 / 362880.0;
    p = p * r + 1.0 / 40320.0;
    p = p * r + 1.0 / 5040.0;
    p = p * r + 1.0 / 720.0;
    p = p * r + 1.0 / 120.0;
    p = p * r + 1.0 / 24.0;
    p = p * r + 1.0 / 6.0;
    p = p * r + 0.5;
    p = p * r + 1.0;
    p = p * r + 1.0;
    const int64_t k = static_cast<int64_t>(kd);
    uint64_t bits = static_cast<uint64_t>(k + 1023) << 52;
    double two_k;
    std::memcpy(&two_k, &bits, 8);
    return static_cast<float>(p * two_k);
}

uint64_t orc_mix64(uint64_t a, uint64_t b) {
    // restates mix64, src/dataset.cpp:11-17
    uint64_t z = a ^ (b + 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

int orc_has_nonfinite(const float* g, int64_t n) {
    // src/trainer.cpp:78-82
    for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(g[i])) return 1;
    return 0;
}

void orc_apply_sgd(float* w, float* v, const float* gsum, int64_t n, float lr, float mu, double denom) {
    // src/trainer.cpp:86-94, verbatim arithmetic order
    const float inv = static_cast<float>(1.0 / denom);
    for (int64_t i = 0; i < n; ++i) {
        const float g = gsum[i] * inv;
        v[i] = mu * v[i] + g;
        w[i] -= lr * v[i];
    }
}

void orc_update_scale(double* scale, int64_t* good_steps, int dynamic, int64_t growth_interval,
                      double growth, double backoff, double min_scale, double max_scale, int overflow) {
    // src/precision.cpp:45-56
    if (!dynamic) return;
    if (overflow) {
        *scale = std::max(min_scale, *scale * backoff);
        *good_steps = 0;
        return;
    }
    if (++*good_steps >= growth_interval) {
        *scale = std::min(max_scale, *scale * growth);
        *good_steps = 0;
    }
}

double orc_softmax_ce(const float* ld, int64_t B, int64_t C, const int32_t* lab, double dy, double grad_scale,
                      float* dx) {
    // src/model.cpp:106-150: FP64 max/logsumexp, probabilities stored as
    // float, loss = mean(-log p_y), dx = (p - onehot) * (dy*grad_scale/B)
    std::vector<float> pd(static_cast<size_t>(B * C));
    double loss = 0.0;
    for (int64_t i = 0; i < B; ++i) {
        double mx = ld[i * C];
        for (int64_t j = 1; j < C; ++j) mx = std::max(mx, static_cast<double>(ld[i * C + j]));
        double z = 0.0;
        for (int64_t j = 0; j < C; ++j) z += std::exp(static_cast<double>(ld[i * C + j]) - mx);
        for (int64_t j = 0; j < C; ++j)
            pd[i * C + j] = static_cast<float>(std::exp(static_cast<double>(ld[i * C + j]) - mx) / z);
        loss -= std::log(std::max(1e-30, static_cast<double>(pd[i * C + lab[i]])));
    }
    if (dx) {
        const float g = static_cast<float>(dy * grad_scale / static_cast<double>(B));
        for (int64_t i = 0; i < B; ++i)
            for (int64_t j = 0; j < C; ++j) dx[i * C + j] = (pd[i * C + j] - (j == lab[i] ? 1.0f : 0.0f)) * g;
    }
    return loss / static_cast<double>(B);
}

double orc_sigmoid_bce(const float* x, const int8_t* lab, int64_t n, double norm, double grad_scale, float* dx) {
    double loss = 0.0;
    const double gs = grad_scale / norm;
    for (int64_t i = 0; i < n; ++i) {
        if (lab[i] < 0) {
            if (dx) dx[i] = 0.0f;
            continue;
        }
        const double v = x[i], t = lab[i];
        loss += std::max(v, 0.0) - v * t + std::log1p(std::exp(-std::fabs(v)));
        if (dx) {
            const double s = 1.0 / (1.0 + std::exp(-v));
            dx[i] = static_cast<float>((s - t) * gs);
        }
    }
    return loss / norm;
}

double orc_smooth_l1(const float* pred, const float* target, const float* weight, int64_t rows, double beta,
                     double norm, double grad_scale, float* dpred) {
    double loss = 0.0;
    const double gs = grad_scale / norm;
    for (int64_t i = 0; i < rows; ++i)
        for (int k = 0; k < 4; ++k) {
            const int64_t at = i * 4 + k;
            if (weight[i] == 0.0f) {
                if (dpred) dpred[at] = 0.0f;
                continue;
            }
            const double d = static_cast<double>(pred[at]) - static_cast<double>(target[at]);
            const double ad = std::fabs(d);
            loss += weight[i] * (ad < beta ? 0.5 * d * d / beta : ad - 0.5 * beta);
            if (dpred) {
                const double g = ad < beta ? d / beta : (d > 0 ? 1.0 : -1.0);
                dpred[at] = static_cast<float>(weight[i] * g * gs);
            }
        }
    return loss / norm;
}

double orc_iou(const float* a, const float* b) { return iou_d(widen(a), widen(b)); }

void orc_anchors(int H, int W, float stride, const float* scales, int ns, const float* ratios, int nr, float* out) {
    const int A = ns * nr;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int i = 0; i < nr; ++i)
                for (int j = 0; j < ns; ++j) {
                    const int64_t a = (static_cast<int64_t>(y) * W + x) * A + i * ns + j;
                    const float cx = (static_cast<float>(x) + 0.5f) * stride;
                    const float cy = (static_cast<float>(y) + 0.5f) * stride;
                    const double sr = std::sqrt(static_cast<double>(ratios[i]));
                    const float w = static_cast<float>(static_cast<double>(scales[j]) / sr);
                    const float h = static_cast<float>(static_cast<double>(scales[j]) * sr);
                    out[a * 4 + 0] = cx - 0.5f * w;
                    out[a * 4 + 1] = cy - 0.5f * h;
                    out[a * 4 + 2] = cx + 0.5f * w;
                    out[a * 4 + 3] = cy + 0.5f * h;
                }
}

void orc_decode(const float* an, const float* d, int64_t n, const float* wt, float clip_dw, float img_h,
                float img_w, float* out) {
    for (int64_t i = 0; i < n; ++i) {
        const float* a = an + i * 4;
        const float aw = a[2] - a[0], ah = a[3] - a[1];
        const float acx = a[0] + 0.5f * aw, acy = a[1] + 0.5f * ah;
        const float dx = d[i * 4 + 0] / wt[0], dy = d[i * 4 + 1] / wt[1];
        const float dw = std::min(d[i * 4 + 2] / wt[2], clip_dw);
        const float dh = std::min(d[i * 4 + 3] / wt[3], clip_dw);
        const float pcx = dx * aw + acx, pcy = dy * ah + acy;
        const float pw = orc_expf(dw) * aw, ph = orc_expf(dh) * ah;
        out[i * 4 + 0] = std::min(std::max(pcx - 0.5f * pw, 0.0f), img_w);
        out[i * 4 + 1] = std::min(std::max(pcy - 0.5f * ph, 0.0f), img_h);
        out[i * 4 + 2] = std::min(std::max(pcx + 0.5f * pw, 0.0f), img_w);
        out[i * 4 + 3] = std::min(std::max(pcy + 0.5f * ph, 0.0f), img_h);
    }
}

void orc_encode(const float* ex, const float* gt, int64_t n, const float* wt, float* t) {
    for (int64_t i = 0; i < n; ++i) {
        const float* e = ex + i * 4;
        const float* g = gt + i * 4;
        const float ew = e[2] - e[0], eh = e[3] - e[1];
        const float ecx = e[0] + 0.5f * ew, ecy = e[1] + 0.5f * eh;
        const float gw = g[2] - g[0], gh = g[3] - g[1];
        const float gcx = g[0] + 0.5f * gw, gcy = g[1] + 0.5f * gh;
        t[i * 4 + 0] = wt[0] * (gcx - ecx) / ew;
        t[i * 4 + 1] = wt[1] * (gcy - ecy) / eh;
        t[i * 4 + 2] = wt[2] * std::log(gw / ew);
        t[i * 4 + 3] = wt[3] * std::log(gh / eh);
    }
}

void orc_topk_order(const float* s, int64_t n, int64_t k, int32_t* order) {
    // std::stable_sort by score desc keeps index-asc among ties
    // (src/postproc.cpp:41-43); NaN is ranked below -inf.
    std::vector<int32_t> idx(static_cast<size_t>(n));
    std::iota(idx.begin(), idx.end(), 0);
    auto key = [&](int32_t i) {
        const float v = s[i];
        return v != v ? -std::numeric_limits<double>::infinity() : static_cast<double>(v);
    };
    std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
        const float va = s[a], vb = s[b];
        const bool na = va != va, nb = vb != vb;
        if (na != nb) return nb;  // non-NaN first
        if (na) return false;
        return key(a) > key(b);
    });
    for (int64_t i = 0; i < k && i < n; ++i) order[i] = idx[static_cast<size_t>(i)];
}

int64_t orc_nms_sorted(const float* boxes, int64_t n, double thr, int64_t max_keep, int32_t* keep) {
    // greedy keep/suppress of src/postproc.cpp:47-63 over a pre-sorted list
    std::vector<char> dead(static_cast<size_t>(n), 0);
    int64_t k = 0;
    for (int64_t i = 0; i < n && k < max_keep; ++i) {
        if (dead[i]) continue;
        keep[k++] = static_cast<int32_t>(i);
        const BoxD bi = widen(boxes + i * 4);
        for (int64_t j = i + 1; j < n; ++j)
            if (!dead[j] && iou_d(bi, widen(boxes + j * 4)) > thr) dead[j] = 1;
    }
    return k;
}

int64_t orc_proposals(const float* logits, const float* deltas, const float* anchors, int64_t nA, float img_h,
                      float img_w, int64_t pre_k, double iou, int64_t post_k, float* rois, float* roi_scores,
                      int32_t* topk_order) {
    const int64_t k = std::min(pre_k, nA);
    std::vector<int32_t> order(static_cast<size_t>(k));
    orc_topk_order(logits, nA, k, order.data());
    if (topk_order) std::copy(order.begin(), order.end(), topk_order);
    std::vector<float> an(static_cast<size_t>(k * 4)), dl(static_cast<size_t>(k * 4)), bx(static_cast<size_t>(k * 4));
    for (int64_t i = 0; i < k; ++i)
        for (int c = 0; c < 4; ++c) {
            an[i * 4 + c] = anchors[static_cast<int64_t>(order[i]) * 4 + c];
            dl[i * 4 + c] = deltas[static_cast<int64_t>(order[i]) * 4 + c];
        }
    const float one[4] = {1.0f, 1.0f, 1.0f, 1.0f};
    const float clip = static_cast<float>(std::log(1000.0 / 16.0));
    orc_decode(an.data(), dl.data(), k, one, clip, img_h, img_w, bx.data());
    std::vector<int32_t> keep(static_cast<size_t>(std::max<int64_t>(post_k, 1)));
    const int64_t nk = orc_nms_sorted(bx.data(), k, iou, post_k, keep.data());
    for (int64_t i = 0; i < nk; ++i) {
        for (int c = 0; c < 4; ++c) rois[i * 4 + c] = bx[static_cast<int64_t>(keep[i]) * 4 + c];
        if (roi_scores) roi_scores[i] = logits[order[keep[i]]];
    }
    return nk;
}

void orc_anchor_targets(const float* anchors, int64_t nA, const float* gt, int64_t G, float img_h, float img_w,
                        uint64_t key, double fg_thr, double bg_thr, int64_t batch, double fg_frac, int8_t* labels,
                        float* bbox_targets) {
    std::vector<double> max_iou(static_cast<size_t>(nA), -1.0), gt_max(static_cast<size_t>(G), 0.0);
    std::vector<int32_t> arg(static_cast<size_t>(nA), 0);
    std::vector<char> inside(static_cast<size_t>(nA), 0);
    for (int64_t a = 0; a < nA; ++a) {
        labels[a] = -1;
        const float* b = anchors + a * 4;
        inside[a] = b[0] >= 0.0f && b[1] >= 0.0f && b[2] <= img_w && b[3] <= img_h;
        if (!inside[a]) continue;
        const BoxD ab = widen(b);
        double best = 0.0;
        int32_t bi = 0;
        for (int64_t g = 0; g < G; ++g) {
            const double v = iou_d(ab, widen(gt + g * 4));
            if (v > best) { best = v; bi = static_cast<int32_t>(g); }
            if (v > gt_max[g]) gt_max[g] = v;
        }
        max_iou[a] = best;
        arg[a] = bi;
    }
    for (int64_t a = 0; a < nA; ++a)
        if (inside[a] && max_iou[a] < bg_thr) labels[a] = 0;
    for (int64_t a = 0; a < nA; ++a) {
        if (!inside[a]) continue;
        const BoxD ab = widen(anchors + a * 4);
        for (int64_t g = 0; g < G; ++g)
            if (gt_max[g] > 0.0 && iou_d(ab, widen(gt + g * 4)) == gt_max[g]) { labels[a] = 1; break; }
        if (max_iou[a] >= fg_thr) labels[a] = 1;
    }
    std::vector<int64_t> fg, bg;
    for (int64_t a = 0; a < nA; ++a) {
        if (labels[a] == 1) fg.push_back(a);
        else if (labels[a] == 0) bg.push_back(a);
    }
    const int64_t cap = static_cast<int64_t>(fg_frac * static_cast<double>(batch));
    if (static_cast<int64_t>(fg.size()) > cap) {
        const auto keepv = pick_smallest(fg, key, cap);
        for (int64_t a : fg) labels[a] = -1;
        for (int64_t a : keepv) labels[a] = 1;
        fg = keepv;
    }
    const int64_t nbg = batch - static_cast<int64_t>(fg.size());
    if (static_cast<int64_t>(bg.size()) > nbg) {
        const auto keepv = pick_smallest(bg, orc_mix64(key, 0xb9ull), nbg);
        for (int64_t a : bg) labels[a] = -1;
        for (int64_t a : keepv) labels[a] = 0;
    }
    const float one[4] = {1.0f, 1.0f, 1.0f, 1.0f};
    for (int64_t a = 0; a < nA; ++a) {
        float* t = bbox_targets + a * 4;
        t[0] = t[1] = t[2] = t[3] = 0.0f;
        if (labels[a] == 1 && G > 0) orc_encode(anchors + a * 4, gt + static_cast<int64_t>(arg[a]) * 4, 1, one, t);
    }
}

int64_t orc_proposal_targets(const float* rois, int64_t R, const float* gt, const int32_t* gt_cls, int64_t G,
                             uint64_t key, double fg_thr, double bg_hi, double bg_lo, int64_t batch, double fg_frac,
                             float* out_rois, int32_t* out_labels, float* out_targets, int32_t* out_src) {
    const int64_t T = R + G;  // proposals followed by the ground truth boxes
    auto cand = [&](int64_t i) { return i < R ? rois + i * 4 : gt + (i - R) * 4; };
    std::vector<double> mx(static_cast<size_t>(T), 0.0);
    std::vector<int32_t> arg(static_cast<size_t>(T), 0);
    std::vector<int64_t> fg, bg;
    for (int64_t i = 0; i < T; ++i) {
        const BoxD b = widen(cand(i));
        double best = 0.0;
        int32_t bi = 0;
        for (int64_t g = 0; g < G; ++g) {
            const double v = iou_d(b, widen(gt + g * 4));
            if (v > best) { best = v; bi = static_cast<int32_t>(g); }
        }
        mx[i] = best;
        arg[i] = bi;
        if (G > 0 && best >= fg_thr) fg.push_back(i);
        else if (best < bg_hi && best >= bg_lo) bg.push_back(i);
    }
    const int64_t fg_cap = static_cast<int64_t>(std::llround(fg_frac * static_cast<double>(batch)));
    const auto fgk = pick_smallest(fg, key, std::min<int64_t>(fg_cap, static_cast<int64_t>(fg.size())));
    const int64_t nbg = std::min<int64_t>(batch - static_cast<int64_t>(fgk.size()), static_cast<int64_t>(bg.size()));
    const auto bgk = pick_smallest(bg, orc_mix64(key, 0xb9ull), nbg);
    const float w[4] = {10.0f, 10.0f, 5.0f, 5.0f};
    int64_t s = 0;
    for (int pass = 0; pass < 2; ++pass) {
        const auto& v = pass == 0 ? fgk : bgk;
        for (int64_t i : v) {
            const float* b = cand(i);
            for (int c = 0; c < 4; ++c) out_rois[s * 4 + c] = b[c];
            out_labels[s] = pass == 0 ? gt_cls[arg[i]] : 0;
            float* t = out_targets + s * 4;
            t[0] = t[1] = t[2] = t[3] = 0.0f;
            if (pass == 0) orc_encode(b, gt + static_cast<int64_t>(arg[i]) * 4, 1, w, t);
            if (out_src) out_src[s] = static_cast<int32_t>(i);
            ++s;
        }
    }
    return s;
}

void orc_roialign_fwd(const float* feat, int N, int C, int H, int W, const float* rois, int64_t R, int P,
                      float scale, int sr, int aligned, float* out) {
    (void)N;
    const float count = static_cast<float>(std::max(sr * sr, 1));
    for (int64_t r = 0; r < R; ++r) {
        const RoiGeom g = roi_geom(rois + r * 5, P, scale, aligned);
        for (int c = 0; c < C; ++c) {
            const float* f = feat + (static_cast<int64_t>(g.b) * C + c) * H * W;
            for (int ph = 0; ph < P; ++ph)
                for (int pw = 0; pw < P; ++pw) {
                    float acc = 0.0f;
                    for (int iy = 0; iy < sr; ++iy) {
                        const float y = g.sh + static_cast<float>(ph) * g.bh +
                                        (static_cast<float>(iy) + 0.5f) * g.bh / static_cast<float>(sr);
                        for (int ix = 0; ix < sr; ++ix) {
                            const float x = g.sw + static_cast<float>(pw) * g.bw +
                                            (static_cast<float>(ix) + 0.5f) * g.bw / static_cast<float>(sr);
                            acc += bilinear(f, H, W, y, x);
                        }
                    }
                    out[((r * C + c) * P + ph) * P + pw] = acc / count;
                }
        }
    }
}

void orc_roialign_bwd(const float* dy, int N, int C, int H, int W, const float* rois, int64_t R, int P,
                      float scale, int sr, int aligned, float* dfeat) {
    std::fill(dfeat, dfeat + static_cast<int64_t>(N) * C * H * W, 0.0f);
    const float count = static_cast<float>(std::max(sr * sr, 1));
    for (int64_t r = 0; r < R; ++r) {
        const RoiGeom g = roi_geom(rois + r * 5, P, scale, aligned);
        for (int c = 0; c < C; ++c) {
            float* f = dfeat + (static_cast<int64_t>(g.b) * C + c) * H * W;
            for (int ph = 0; ph < P; ++ph)
                for (int pw = 0; pw < P; ++pw) {
                    const float gv = dy[((r * C + c) * P + ph) * P + pw];
                    for (int iy = 0; iy < sr; ++iy) {
                        const float y = g.sh + static_cast<float>(ph) * g.bh +
                                        (static_cast<float>(iy) + 0.5f) * g.bh / static_cast<float>(sr);
                        for (int ix = 0; ix < sr; ++ix) {
                            const float x = g.sw + static_cast<float>(pw) * g.bw +
                                            (static_cast<float>(ix) + 0.5f) * g.bw / static_cast<float>(sr);
                            const Corner k = corners(H, W, y, x);
                            if (!k.valid) continue;
                            f[k.yl * W + k.xl] += gv * k.w1 / count;
                            f[k.yl * W + k.xh] += gv * k.w2 / count;
                            f[k.yh * W + k.xl] += gv * k.w3 / count;
                            f[k.yh * W + k.xh] += gv * k.w4 / count;
                        }
                    }
                }
        }
    }
}

void orc_maxpool_fwd(const float* x, int N, int C, int H, int W, int k, int s, int p, float* y) {
    const int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
    for (int64_t nc = 0; nc < static_cast<int64_t>(N) * C; ++nc)
        for (int oh = 0; oh < Ho; ++oh)
            for (int ow = 0; ow < Wo; ++ow) {
                float m = -std::numeric_limits<float>::infinity();
                for (int r = 0; r < k; ++r)
                    for (int q = 0; q < k; ++q) {
                        const int ih = oh * s - p + r, iw = ow * s - p + q;
                        if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
                        const float v = x[(nc * H + ih) * W + iw];
                        if (v > m) m = v;
                    }
                y[(nc * Ho + oh) * Wo + ow] = m;
            }
}

void orc_maxpool_bwd(const float* x, const float* dy, int N, int C, int H, int W, int k, int s, int p, float* dx) {
    // gradient goes to the first maximum in (r, q) scan order
    const int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
    std::fill(dx, dx + static_cast<int64_t>(N) * C * H * W, 0.0f);
    for (int64_t nc = 0; nc < static_cast<int64_t>(N) * C; ++nc)
        for (int oh = 0; oh < Ho; ++oh)
            for (int ow = 0; ow < Wo; ++ow) {
                float m = -std::numeric_limits<float>::infinity();
                int64_t at = -1;
                for (int r = 0; r < k; ++r)
                    for (int q = 0; q < k; ++q) {
                        const int ih = oh * s - p + r, iw = ow * s - p + q;
                        if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
                        const int64_t i = (nc * H + ih) * W + iw;
                        if (at < 0 || x[i] > m) { m = x[i]; at = i; }
                    }
                dx[at] += dy[(nc * Ho + oh) * Wo + ow];
            }
}

void orc_avgpool_fwd(const float* x, int N, int C, int H, int W, float* y) {
    for (int64_t nc = 0; nc < static_cast<int64_t>(N) * C; ++nc) {
        float acc = 0.0f;
        for (int64_t i = 0; i < static_cast<int64_t>(H) * W; ++i) acc += x[nc * H * W + i];
        y[nc] = acc / static_cast<float>(H * W);
    }
}

void orc_avgpool_bwd(const float* dy, int N, int C, int H, int W, float* dx) {
    for (int64_t nc = 0; nc < static_cast<int64_t>(N) * C; ++nc)
        for (int64_t i = 0; i < static_cast<int64_t>(H) * W; ++i) dx[nc * H * W + i] = dy[nc] / static_cast<float>(H * W);
}

// ---- SyncBN over K ranks (TEST-ONLY restatement).
// CommGroup::allreduce_sum (src/comm.cpp:230-240, 288-315): ring reduce-scatter
// over ring_chunks(n, K); the element of chunk c is left-folded in rank order
// c, c+1, ..., c+K-1 (mod K), then all-gathered, so every rank holds the same
// bits.  bufs = [K][n], reduced in place.
void orc_ring_allreduce_sum(float* bufs, int K, int64_t n) {
    if (K <= 1) return;
    const int64_t base = n / K, rem = n % K;
    int64_t at = 0;
    for (int c = 0; c < K; ++c) {
        const int64_t len = base + (c < rem ? 1 : 0);
        for (int64_t i = at; i < at + len; ++i) {
            float acc = bufs[static_cast<int64_t>(c) * n + i];
            for (int j = 1; j < K; ++j) acc = acc + bufs[static_cast<int64_t>((c + j) % K) * n + i];
            for (int r = 0; r < K; ++r) bufs[static_cast<int64_t>(r) * n + i] = acc;
        }
        at += len;
    }
}

// syncbn_forward with a K-rank group (src/syncbn.cpp:21-70): x_all = [K][N][C][H][W]
// (each rank's shard, NCHW); y_all likewise; mean/invstd/agg are the (identical)
// per-rank results; agg = [sum, sumsq, count] after the allreduce.  fp16: the
// output is rounded to binary16 (Tensor::quantize).
void orc_syncbn_forward_k(int K, const float* x_all, int N, int C, int H, int W, const float* gamma,
                          const float* beta, float eps, int fp16, float* y_all, float* mean, float* invstd,
                          float* agg) {
    const int64_t hw = static_cast<int64_t>(H) * W, per = static_cast<int64_t>(N) * C * hw, n = 2 * C + 1;
    std::vector<float> bufs(static_cast<size_t>(K) * n, 0.0f);
    for (int r = 0; r < K; ++r) {
        const float* xd = x_all + r * per;
        float* a = bufs.data() + static_cast<int64_t>(r) * n;
        for (int c = 0; c < C; ++c) {
            double s = 0.0, sq = 0.0;
            for (int b = 0; b < N; ++b)
                for (int64_t i = 0; i < hw; ++i) {
                    const double v = xd[(static_cast<int64_t>(b) * C + c) * hw + i];
                    s += v;
                    sq += v * v;
                }
            a[c] = static_cast<float>(s);
            a[C + c] = static_cast<float>(sq);
        }
        a[2 * C] = static_cast<float>(static_cast<int64_t>(N) * hw);
    }
    orc_ring_allreduce_sum(bufs.data(), K, n);
    const float* g = bufs.data();
    std::memcpy(agg, g, static_cast<size_t>(n) * sizeof(float));
    const int64_t count = static_cast<int64_t>(g[2 * C]);
    for (int c = 0; c < C; ++c) {
        const double mu = static_cast<double>(g[c]) / count;
        double var = static_cast<double>(g[C + c]) / count - mu * mu;
        if (var < 0.0) var = 0.0;
        mean[c] = static_cast<float>(mu);
        invstd[c] = static_cast<float>(1.0 / std::sqrt(var + eps));
    }
    for (int r = 0; r < K; ++r)
        for (int b = 0; b < N; ++b)
            for (int c = 0; c < C; ++c)
                for (int64_t i = 0; i < hw; ++i) {
                    const int64_t at = r * per + (static_cast<int64_t>(b) * C + c) * hw + i;
                    const float v = gamma[c] * (x_all[at] - mean[c]) * invstd[c] + beta[c];
                    y_all[at] = fp16 ? orc_half_round(v) : v;
                }
}

// syncbn_backward with a K-rank group (src/syncbn.cpp:72-117); count = the
// forward's GLOBAL count; dgamma/dbeta = the all-reduced sums
void orc_syncbn_backward_k(int K, const float* dy_all, const float* x_all, int N, int C, int H, int W,
                           const float* gamma, const float* mean, const float* invstd, int64_t count, float* dx_all,
                           float* dgamma, float* dbeta) {
    const int64_t hw = static_cast<int64_t>(H) * W, per = static_cast<int64_t>(N) * C * hw, n = 2 * C;
    std::vector<float> bufs(static_cast<size_t>(K) * n, 0.0f);
    for (int r = 0; r < K; ++r) {
        const float* xd = x_all + r * per;
        const float* gd = dy_all + r * per;
        float* red = bufs.data() + static_cast<int64_t>(r) * n;
        for (int c = 0; c < C; ++c) {
            double s1 = 0.0, s2 = 0.0;
            for (int b = 0; b < N; ++b)
                for (int64_t i = 0; i < hw; ++i) {
                    const int64_t at = (static_cast<int64_t>(b) * C + c) * hw + i;
                    const double xh = (xd[at] - mean[c]) * invstd[c];
                    s1 += gd[at];
                    s2 += gd[at] * xh;
                }
            red[c] = static_cast<float>(s1);
            red[C + c] = static_cast<float>(s2);
        }
    }
    orc_ring_allreduce_sum(bufs.data(), K, n);
    const float* red = bufs.data();
    const float m = static_cast<float>(count);
    for (int c = 0; c < C; ++c) {
        dgamma[c] = red[C + c];
        dbeta[c] = red[c];
    }
    for (int r = 0; r < K; ++r)
        for (int b = 0; b < N; ++b)
            for (int c = 0; c < C; ++c) {
                const float gis = gamma[c] * invstd[c];
                const float s1 = red[c] / m, s2 = red[C + c] / m;
                for (int64_t i = 0; i < hw; ++i) {
                    const int64_t at = r * per + (static_cast<int64_t>(b) * C + c) * hw + i;
                    const float xh = (x_all[at] - mean[c]) * invstd[c];
                    dx_all[at] = gis * (dy_all[at] - s1 - xh * s2);
                }
            }
}

}  // extern "C"
