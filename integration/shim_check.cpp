// integration/shim_check.cpp -- TEST VENEER ONLY: extern "C" entry points that
// build reference Tensors from raw arrays, call the simdet::gpu shim
// (simdet_gpu.hpp) exactly as a simdet caller would, and return raw arrays,
// so tests/test_gpu_integration.py can hold the shim against the reference
// engine's own CPU functions (oracle/_ref).  Status codes follow
// oracle/ref_capi.cpp (the reference exception taxonomy).
#include <cstring>
#include <string>
#include <vector>

#include "simdet/errors.hpp"
#include "simdet_gpu.hpp"

using namespace simdet;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 1;
    } catch (const ContractError& e) {
        g_err = e.what();
        return 2;
    } catch (const DegenerateBatchError& e) {
        g_err = e.what();
        return 3;
    } catch (const NonInvertibleError& e) {
        g_err = e.what();
        return 4;
    } catch (const ParamError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 99;
    }
}

Tensor mk(std::vector<int64_t> s, int fp16, const float* p) {
    int64_t n = 1;
    for (int64_t d : s) n *= d;
    return Tensor(std::move(s), fp16 ? DType::F16 : DType::F32, std::vector<float>(p, p + n));
}

void put(const Tensor& t, float* out) { std::memcpy(out, t.data().data(), t.data().size() * sizeof(float)); }
void putv(const std::vector<float>& v, float* out) { std::memcpy(out, v.data(), v.size() * sizeof(float)); }
}  // namespace

extern "C" {

const char* shim_last_error() { return g_err.c_str(); }

int shim_conv2d(const float* x, int N, int C, int H, int W, const float* k, int O, int kh, int kw, int stride, int pad,
                int fp16, float* y) {
    return guarded([&] { put(gpu::conv2d(mk({N, C, H, W}, fp16, x), mk({O, C, kh, kw}, fp16, k), stride, pad), y); });
}

int shim_conv2d_backward(const float* x, int N, int C, int H, int W, const float* k, int O, int kh, int kw,
                         int stride, int pad, int fp16, const float* dy, float* dx, float* dk) {
    return guarded([&] {
        const Tensor xt = mk({N, C, H, W}, fp16, x), kt = mk({O, C, kh, kw}, fp16, k);
        const Shape os = conv2d_out_shape(xt.shape(), kt.shape(), stride, pad);
        auto [gx, gk] = gpu::conv2d_backward(xt, kt, mk(os, 0, dy), stride, pad);
        put(gx, dx);
        put(gk, dk);
    });
}

int shim_bn_forward(const float* x, int N, int C, int H, int W, const float* gamma, const float* beta, float eps,
                    int fp16, float* y, float* mean, float* invstd, float* sum, float* sumsq, int64_t* count) {
    return guarded([&] {
        auto [yt, st] = gpu::syncbn_forward(mk({N, C, H, W}, fp16, x), std::span<const float>(gamma, C),
                                            std::span<const float>(beta, C), eps, nullptr);
        put(yt, y);
        putv(st.mean, mean);
        putv(st.invstd, invstd);
        putv(st.sum, sum);
        putv(st.sumsq, sumsq);
        *count = st.count;
    });
}

int shim_bn_backward(const float* dy, const float* x, int N, int C, int H, int W, const float* gamma,
                     const float* mean, const float* invstd, int fp16, float* dx, float* dgamma, float* dbeta) {
    return guarded([&] {
        BNStats st;
        st.count = static_cast<int64_t>(N) * H * W;
        st.mean.assign(mean, mean + C);
        st.invstd.assign(invstd, invstd + C);
        BnGrads g = gpu::syncbn_backward(mk({N, C, H, W}, 0, dy), mk({N, C, H, W}, fp16, x), st,
                                         std::span<const float>(gamma, C), nullptr);
        put(g.dx, dx);
        putv(g.dgamma, dgamma);
        putv(g.dbeta, dbeta);
    });
}

int shim_iabn_forward(const float* x, int N, int C, int H, int W, const float* gamma, const float* beta, float eps,
                      float slope, int fp16, float* y, float* mean, float* invstd) {
    return guarded([&] {
        auto [yt, sv] = gpu::iabn_forward(mk({N, C, H, W}, fp16, x), std::span<const float>(gamma, C),
                                          std::span<const float>(beta, C), eps, slope);
        put(yt, y);
        putv(sv.mean, mean);
        putv(sv.invstd, invstd);
    });
}

int shim_iabn_backward(const float* dy, const float* y, int N, int C, int H, int W, const float* gamma,
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
        IabnGrads g = gpu::iabn_backward(mk({N, C, H, W}, 0, dy), sv);
        put(g.dx, dx);
        putv(g.dgamma, dgamma);
        putv(g.dbeta, dbeta);
    });
}

int shim_apply_sgd(float* w, float* v, const float* g, int64_t n, float lr, float mu, double scale, int K,
                   int* skipped) {
    return guarded([&] {
        *skipped = gpu::apply_sgd(std::span<float>(w, n), std::span<float>(v, n), std::span<const float>(g, n), lr, mu,
                                  scale, K)
                       ? 1
                       : 0;
    });
}

}  // extern "C"
