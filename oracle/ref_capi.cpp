// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" veneer over the UNMODIFIED reference engine `simdet`
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libsimdet_ref.so).  Lets the Python tests call the reference's
// own conv2d / BN / IABN / matmul / NMS / binary16 / loss-scale code on the
// same seeded inputs the CUDA path sees.  Nothing here is product code.
//
// Status codes mirror the reference's exception taxonomy (errors.hpp:9-40) the
// same way include/sdb.h does, so error-behaviour parity can be asserted.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "simdet/autograd.hpp"
#include "simdet/checkpoint.hpp"
#include "simdet/comm.hpp"
#include "simdet/errors.hpp"
#include "simdet/half.hpp"
#include "simdet/memopt.hpp"
#include "simdet/postproc.hpp"
#include "simdet/precision.hpp"
#include "simdet/syncbn.hpp"
#include "simdet/tensor.hpp"

using namespace simdet;

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ShapeError*>(&e)) return 1;
    if (dynamic_cast<const ContractError*>(&e)) return 2;
    if (dynamic_cast<const DegenerateBatchError*>(&e)) return 3;
    if (dynamic_cast<const NonInvertibleError*>(&e)) return 4;
    if (dynamic_cast<const ParamError*>(&e)) return 5;
    if (dynamic_cast<const CollectiveError*>(&e)) return 6;
    return 99;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

inline DType dt(int fp16) { return fp16 ? DType::F16 : DType::F32; }

Tensor mk(std::vector<int64_t> shape, int fp16, const float* p) {
    int64_t n = 1;
    for (int64_t d : shape) n *= d;
    return Tensor(std::move(shape), dt(fp16), std::vector<float>(p, p + n));
}

void put(const Tensor& t, float* out) { std::memcpy(out, t.data().data(), t.data().size() * sizeof(float)); }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint16_t ref_float_to_half_bits(float f) { return float_to_half_bits(f); }
float ref_half_bits_to_float(uint16_t h) { return half_bits_to_float(h); }

// simdet::conv2d, src/tensor.cpp:169-196
int ref_conv2d(const float* x, int N, int C, int H, int W, const float* k, int O, int kh, int kw, int stride, int pad,
               int fp16, float* y) {
    return guarded([&] {
        Tensor out = conv2d(mk({N, C, H, W}, fp16, x), mk({O, C, kh, kw}, fp16, k), stride, pad);
        put(out, y);
    });
}

// conv2d backward through the reference tape, src/autograd.cpp:290-320 and the
// dtype finalisation of run_backward (src/autograd.cpp:437-440,475-485)
int ref_conv2d_backward(const float* x, int N, int C, int H, int W, const float* k, int O, int kh, int kw, int stride,
                        int pad, int fp16, const float* dy, float* dx, float* dk) {
    return guarded([&] {
        Tape t;
        ValueId xv = t.leaf(mk({N, C, H, W}, fp16, x));
        ValueId kv = t.leaf(mk({O, C, kh, kw}, fp16, k));
        ValueId yv = t.conv2d(xv, kv, stride, pad);
        const Shape ys = t.value(yv).shape();
        GradMap g = t.backward_from(yv, mk(ys, 0, dy));
        put(g.at(xv), dx);
        put(g.at(kv), dk);
    });
}

// simdet::matmul forward + backward (src/tensor.cpp:135-155, src/autograd.cpp:269-289)
int ref_matmul(const float* a, int M, int K, const float* b, int Nn, int fp16, const float* dy, float* y, float* da,
               float* db) {
    return guarded([&] {
        Tape t;
        ValueId av = t.leaf(mk({M, K}, fp16, a));
        ValueId bv = t.leaf(mk({K, Nn}, fp16, b));
        ValueId yv = t.matmul(av, bv);
        put(t.value(yv), y);
        if (dy) {
            GradMap g = t.backward_from(yv, mk({M, Nn}, 0, dy));
            put(g.at(av), da);
            put(g.at(bv), db);
        }
    });
}

// syncbn_forward with group == nullptr (plain BN), src/syncbn.cpp:21-70
int ref_bn_forward(const float* x, int N, int C, int H, int W, const float* gamma, const float* beta, float eps,
                   int fp16, float* y, float* mean, float* invstd) {
    return guarded([&] {
        auto [out, st] = syncbn_forward(mk({N, C, H, W}, fp16, x), std::span<const float>(gamma, C),
                                        std::span<const float>(beta, C), eps, nullptr);
        put(out, y);
        std::memcpy(mean, st.mean.data(), C * sizeof(float));
        std::memcpy(invstd, st.invstd.data(), C * sizeof(float));
    });
}

// syncbn_backward with group == nullptr, src/syncbn.cpp:72-117
int ref_bn_backward(const float* dy, const float* x, int N, int C, int H, int W, const float* gamma,
                    const float* mean, const float* invstd, int fp16, float* dx, float* dgamma, float* dbeta) {
    return guarded([&] {
        BNStats st;
        st.count = static_cast<int64_t>(N) * H * W;
        st.mean.assign(mean, mean + C);
        st.invstd.assign(invstd, invstd + C);
        BnGrads g = syncbn_backward(mk({N, C, H, W}, 0, dy), mk({N, C, H, W}, fp16, x), st,
                                    std::span<const float>(gamma, C), nullptr);
        put(g.dx, dx);
        std::memcpy(dgamma, g.dgamma.data(), C * sizeof(float));
        std::memcpy(dbeta, g.dbeta.data(), C * sizeof(float));
    });
}

// syncbn_forward / syncbn_backward with a K-rank in-process group: the
// reference's own run_workers + CommGroup ring allreduce (src/comm.cpp:242-315).
// x_all/dy_all/y_all/dx_all = [K][N][C][H][W]; mean/invstd/sum/sumsq/count and
// dgamma/dbeta are rank 0's (all ranks agree bitwise).
int ref_syncbn_forward_k(int K, const float* x_all, int N, int C, int H, int W, const float* gamma,
                         const float* beta, float eps, int fp16, float* y_all, float* mean, float* invstd,
                         float* agg) {
    return guarded([&] {
        const int64_t per = static_cast<int64_t>(N) * C * H * W;
        run_workers(K, make_inproc_transport(K), [&](CommGroup& g) {
            const int r = g.rank();
            auto [out, st] = syncbn_forward(mk({N, C, H, W}, fp16, x_all + r * per), std::span<const float>(gamma, C),
                                            std::span<const float>(beta, C), eps, &g);
            put(out, y_all + r * per);
            if (r == 0) {
                std::memcpy(mean, st.mean.data(), C * sizeof(float));
                std::memcpy(invstd, st.invstd.data(), C * sizeof(float));
                std::memcpy(agg, st.sum.data(), C * sizeof(float));
                std::memcpy(agg + C, st.sumsq.data(), C * sizeof(float));
                agg[2 * C] = static_cast<float>(st.count);
            }
        });
    });
}

int ref_syncbn_backward_k(int K, const float* dy_all, const float* x_all, int N, int C, int H, int W,
                          const float* gamma, const float* mean, const float* invstd, int64_t count, int fp16,
                          float* dx_all, float* dgamma, float* dbeta) {
    return guarded([&] {
        const int64_t per = static_cast<int64_t>(N) * C * H * W;
        run_workers(K, make_inproc_transport(K), [&](CommGroup& g) {
            const int r = g.rank();
            BNStats st;
            st.count = count;
            st.mean.assign(mean, mean + C);
            st.invstd.assign(invstd, invstd + C);
            BnGrads gr = syncbn_backward(mk({N, C, H, W}, 0, dy_all + r * per), mk({N, C, H, W}, fp16, x_all + r * per),
                                         st, std::span<const float>(gamma, C), &g);
            put(gr.dx, dx_all + r * per);
            if (r == 0) {
                std::memcpy(dgamma, gr.dgamma.data(), C * sizeof(float));
                std::memcpy(dbeta, gr.dbeta.data(), C * sizeof(float));
            }
        });
    });
}

// load_checkpoint (src/checkpoint.cpp:86-128) of a file written by the GPU
// detector: header fields, the idx-th parameter (name, data) and the velocity
int ref_checkpoint_read(const char* path, int64_t* step, uint64_t* digest, int* nparams, int64_t* nvel,
                        double* scale, int64_t* good, int* mode, int idx, char* name, int name_cap, float* param,
                        int64_t pcap, float* vel, int64_t vcap) {
    return guarded([&] {
        CheckpointState st = load_checkpoint(path);
        *step = st.step;
        *digest = st.config_digest;
        *nparams = static_cast<int>(st.params.size());
        *nvel = static_cast<int64_t>(st.velocity.size());
        *scale = st.scale.scale;
        *good = st.scale.good_steps;
        *mode = st.scale.mode == ScaleMode::Dynamic ? 1 : 0;
        if (idx >= 0 && idx < *nparams) {
            const auto& [nm, t] = st.params[static_cast<size_t>(idx)];
            std::snprintf(name, static_cast<size_t>(name_cap), "%s", nm.c_str());
            const int64_t n = std::min<int64_t>(pcap, t.numel());
            std::memcpy(param, t.data().data(), static_cast<size_t>(n) * sizeof(float));
        }
        const int64_t nv = std::min<int64_t>(vcap, *nvel);
        std::memcpy(vel, st.velocity.data(), static_cast<size_t>(nv) * sizeof(float));
    });
}

// iabn_forward, src/memopt.cpp:226-276
int ref_iabn_forward(const float* x, int N, int C, int H, int W, const float* gamma, const float* beta, float eps,
                     float slope, int fp16, float* y, float* mean, float* invstd) {
    return guarded([&] {
        auto [out, sv] = iabn_forward(mk({N, C, H, W}, fp16, x), std::span<const float>(gamma, C),
                                      std::span<const float>(beta, C), eps, slope);
        put(out, y);
        std::memcpy(mean, sv.mean.data(), C * sizeof(float));
        std::memcpy(invstd, sv.invstd.data(), C * sizeof(float));
    });
}

// iabn_backward, src/memopt.cpp:278-327 (recompute-from-output)
int ref_iabn_backward(const float* dy, const float* y, int N, int C, int H, int W, const float* gamma,
                      const float* beta, const float* mean, const float* invstd, float eps, float slope, int fp16,
                      float* dx, float* dgamma, float* dbeta) {
    return guarded([&] {
        IabnSaved sv;
        sv.y = mk({N, C, H, W}, fp16, y);
        sv.mean.assign(mean, mean + C);
        sv.invstd.assign(invstd, invstd + C);
        sv.gamma.assign(gamma, gamma + C);
        sv.beta.assign(beta, beta + C);
        sv.eps = eps;
        sv.slope = slope;
        IabnGrads g = iabn_backward(mk({N, C, H, W}, 0, dy), sv);
        put(g.dx, dx);
        std::memcpy(dgamma, g.dgamma.data(), C * sizeof(float));
        std::memcpy(dbeta, g.dbeta.data(), C * sizeof(float));
    });
}

// iou / nms_greedy, src/postproc.cpp:20-63
double ref_iou(const double* a, const double* b) {
    Box x{a[0], a[1], a[2], a[3], 1.0, 0}, y{b[0], b[1], b[2], b[3], 1.0, 0};
    return iou(x, y);
}

int ref_nms_greedy(const double* boxes, const double* scores, const int* cls, int64_t n, double thr, int64_t* keep,
                   int64_t* nkeep) {
    return guarded([&] {
        BoxSet bs(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i)
            bs[i] = Box{boxes[i * 4], boxes[i * 4 + 1], boxes[i * 4 + 2], boxes[i * 4 + 3], scores[i], cls ? cls[i] : 0};
        auto k = nms_greedy(bs, thr);
        *nkeep = static_cast<int64_t>(k.size());
        for (size_t i = 0; i < k.size(); ++i) keep[i] = static_cast<int64_t>(k[i]);
    });
}

// update_scale, src/precision.cpp:45-56
int ref_update_scale(double* scale, int64_t* good, int dynamic, int64_t interval, double growth, double backoff,
                     double min_scale, double max_scale, int overflow) {
    return guarded([&] {
        LossScaleState s;
        s.scale = *scale;
        s.good_steps = *good;
        s.mode = dynamic ? ScaleMode::Dynamic : ScaleMode::Static;
        s.growth_interval = interval;
        s.growth_factor = growth;
        s.backoff_factor = backoff;
        s.min_scale = min_scale;
        s.max_scale = max_scale;
        update_scale(s, overflow != 0);
        *scale = s.scale;
        *good = s.good_steps;
    });
}

// CommGroup::allreduce_sum (src/comm.cpp:288-315) over K in-process ranks
// (run_workers, src/comm.cpp:451-471): seconds per call on rank 0, averaged
// over `iters` calls on n floats per rank (the CPU baseline's allreduce term)
int ref_allreduce_seconds(int K, int64_t n, int iters, double* seconds) {
    return guarded([&] {
        auto tr = make_inproc_transport(K);
        double sec = 0.0;
        run_workers(K, tr, [&](CommGroup& g) {
            std::vector<float> buf(static_cast<size_t>(n), 1.0f + static_cast<float>(g.rank()));
            g.allreduce_sum(buf);  // warm-up
            const auto t0 = std::chrono::steady_clock::now();
            for (int i = 0; i < iters; ++i) g.allreduce_sum(buf);
            const auto t1 = std::chrono::steady_clock::now();
            if (g.rank() == 0) sec = std::chrono::duration<double>(t1 - t0).count() / std::max(iters, 1);
        });
        *seconds = sec;
    });
}

// sgd_step_master (src/precision.cpp:84-100): v = mu v + g; w -= lr v
int ref_sgd_step_master(float* w, float* v, const float* g, int64_t n, float lr, float mu) {
    return guarded([&] {
        MasterWeights mw;
        mw.add("p", Tensor({n}, DType::F32, std::vector<float>(w, w + n)));
        auto& p = mw.params.at("p");
        std::memcpy(p.velocity.data().data(), v, n * sizeof(float));
        std::map<std::string, Tensor> gm;
        gm.emplace("p", Tensor({n}, DType::F32, std::vector<float>(g, g + n)));
        sgd_step_master(mw, gm, lr, mu, false);
        std::memcpy(w, p.master.data().data(), n * sizeof(float));
        std::memcpy(v, p.velocity.data().data(), n * sizeof(float));
    });
}

// plan_checkpoints (src/memopt.cpp:76-89): segment boundaries for L layers;
// returns their count (or -1 on PlanError / overflow of cap)
int ref_plan_checkpoints(int64_t L, int64_t* boundaries, int cap) {
    int n = -1;
    const int rc = guarded([&] {
        const CheckpointPlan plan = plan_checkpoints(L);
        if (static_cast<int>(plan.boundaries.size()) > cap) throw std::runtime_error("cap");
        for (size_t i = 0; i < plan.boundaries.size(); ++i) boundaries[i] = plan.boundaries[i];
        n = static_cast<int>(plan.boundaries.size());
    });
    return rc == 0 ? n : -1;
}

}  // extern "C"
