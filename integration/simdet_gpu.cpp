// integration/simdet_gpu.cpp -- see simdet_gpu.hpp.  Compiled against the
// reference headers (/root/reference/proj/include) and include/sdb.h; links
// the reference library (for Tensor, conv2d_out_shape, binary16) and
// libsdb.so.  No CUDA runtime is needed here: device memory goes through the
// sdb_device_* / sdb_copy_* entry points.
#include "simdet_gpu.hpp"

#include <cstdint>
#include <cstring>
#include <string>

#include "../include/sdb.h"
#include "simdet/errors.hpp"
#include "simdet/half.hpp"

namespace simdet::gpu {

namespace {

// sdb_status -> the reference exception taxonomy (errors.hpp:9-40)
[[noreturn]] void raise(int rc) {
    const std::string m = sdb_last_error();
    switch (rc) {
        case SDB_SHAPE: throw ShapeError(m);
        case SDB_CONTRACT: throw ContractError(m);
        case SDB_DEGENERATE: throw DegenerateBatchError(m);
        case SDB_NONINVERTIBLE: throw NonInvertibleError(m);
        case SDB_PARAM: throw ParamError(m);
        case SDB_COLLECTIVE: throw CollectiveError(m);
        case SDB_FORMAT: throw FormatError(m);
        default: throw Error("libsdb: " + m);
    }
}

void ck(int rc) {
    if (rc != SDB_OK) raise(rc);
}

int dt_code(DType d) { return d == DType::F16 ? SDB_F16 : SDB_F32; }

// one device buffer, freed with the context
struct Dev {
    void* p = nullptr;
    size_t bytes = 0;
    explicit Dev(size_t b) : bytes(b) { ck(sdb_device_alloc(context(), b, &p)); }
    ~Dev() { sdb_device_free(context(), p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    float* f() { return static_cast<float*>(p); }
};

// NCHW (or OIHW) float buffer -> device NHWC (KRSC) in the tensor's dtype
void upload_nhwc(const Tensor& t, Dev& d) {
    const Shape& s = t.shape();
    const int64_t N = s[0], C = s[1], H = s.size() > 2 ? s[2] : 1, W = s.size() > 3 ? s[3] : 1;
    const auto src = t.data();
    if (t.dtype() == DType::F16) {
        std::vector<uint16_t> h(static_cast<size_t>(t.numel()));
        for (int64_t n = 0; n < N; ++n)
            for (int64_t c = 0; c < C; ++c)
                for (int64_t y = 0; y < H; ++y)
                    for (int64_t x = 0; x < W; ++x)
                        h[((n * H + y) * W + x) * C + c] = float_to_half_bits(src[((n * C + c) * H + y) * W + x]);
        ck(sdb_copy_to_device(context(), d.p, h.data(), h.size() * 2));
    } else {
        std::vector<float> h(static_cast<size_t>(t.numel()));
        for (int64_t n = 0; n < N; ++n)
            for (int64_t c = 0; c < C; ++c)
                for (int64_t y = 0; y < H; ++y)
                    for (int64_t x = 0; x < W; ++x) h[((n * H + y) * W + x) * C + c] = src[((n * C + c) * H + y) * W + x];
        ck(sdb_copy_to_device(context(), d.p, h.data(), h.size() * 4));
    }
}

// device NHWC in dtype -> NCHW Tensor of `shape` with dtype `out`
Tensor download_nchw(Dev& d, const Shape& shape, DType stored, DType out) {
    const int64_t N = shape[0], C = shape[1], H = shape.size() > 2 ? shape[2] : 1, W = shape.size() > 3 ? shape[3] : 1;
    std::vector<float> v(static_cast<size_t>(N * C * H * W));
    if (stored == DType::F16) {
        std::vector<uint16_t> h(v.size());
        ck(sdb_copy_to_host(context(), h.data(), d.p, h.size() * 2));
        for (int64_t n = 0; n < N; ++n)
            for (int64_t c = 0; c < C; ++c)
                for (int64_t y = 0; y < H; ++y)
                    for (int64_t x = 0; x < W; ++x)
                        v[((n * C + c) * H + y) * W + x] = half_bits_to_float(h[((n * H + y) * W + x) * C + c]);
    } else {
        std::vector<float> h(v.size());
        ck(sdb_copy_to_host(context(), h.data(), d.p, h.size() * 4));
        for (int64_t n = 0; n < N; ++n)
            for (int64_t c = 0; c < C; ++c)
                for (int64_t y = 0; y < H; ++y)
                    for (int64_t x = 0; x < W; ++x) v[((n * C + c) * H + y) * W + x] = h[((n * H + y) * W + x) * C + c];
    }
    return Tensor(shape, out, std::move(v));
}

std::vector<float> download_vec(Dev& d, size_t n) {
    std::vector<float> v(n);
    ck(sdb_copy_to_host(context(), v.data(), d.p, n * 4));
    return v;
}

void upload_vec(std::span<const float> v, Dev& d) { ck(sdb_copy_to_device(context(), d.p, v.data(), v.size() * 4)); }

size_t dev_bytes(const Tensor& t) { return static_cast<size_t>(t.numel()) * (t.dtype() == DType::F16 ? 2 : 4); }

void check_nchw(const Tensor& x, const char* what) {
    if (x.shape().size() != 4) throw ShapeError(std::string(what) + ": rank-4 NCHW tensor required");
}

}  // namespace

sdb_ctx* context() {
    thread_local struct Holder {
        sdb_ctx* c = nullptr;
        ~Holder() {
            if (c) sdb_ctx_destroy(c);
        }
    } h;
    if (!h.c) ck(sdb_ctx_create(0, 0, 1, nullptr, &h.c));
    return h.c;
}

Tensor conv2d(const Tensor& x, const Tensor& k, int stride, int pad) {
    const Shape os = conv2d_out_shape(x.shape(), k.shape(), stride, pad);  // the reference's ShapeErrors
    if (x.dtype() != k.dtype()) throw ShapeError("conv2d: dtype mismatch");
    Dev dx(dev_bytes(x)), dk(dev_bytes(k)), dy(static_cast<size_t>(shape_numel(os)) * (x.dtype() == DType::F16 ? 2 : 4));
    upload_nhwc(x, dx);
    upload_nhwc(k, dk);  // OIHW -> KRSC
    const Shape& s = x.shape();
    ck(sdb_conv_fprop(context(), dt_code(x.dtype()), dx.p, dk.p, dy.p, static_cast<int>(s[0]), static_cast<int>(s[2]),
                      static_cast<int>(s[3]), static_cast<int>(s[1]), static_cast<int>(k.shape()[0]),
                      static_cast<int>(k.shape()[2]), static_cast<int>(k.shape()[3]), stride, pad, nullptr));
    return download_nchw(dy, os, x.dtype(), x.dtype());
}

std::pair<Tensor, Tensor> conv2d_backward(const Tensor& x, const Tensor& k, const Tensor& dy_in, int stride, int pad) {
    const Shape os = conv2d_out_shape(x.shape(), k.shape(), stride, pad);
    if (dy_in.shape() != os) throw ShapeError("conv2d backward: dy shape differs from the output shape");
    const Tensor dy = dy_in.astype(x.dtype());  // incoming gradient in the node's dtype (autograd.cpp:439)
    Dev dxin(dev_bytes(x)), dkin(dev_bytes(k)), ddy(dev_bytes(dy)), ddx(dev_bytes(x)), ddk(dev_bytes(k));
    upload_nhwc(x, dxin);
    upload_nhwc(k, dkin);
    upload_nhwc(dy, ddy);
    const Shape& s = x.shape();
    const int N = static_cast<int>(s[0]), C = static_cast<int>(s[1]), H = static_cast<int>(s[2]),
              W = static_cast<int>(s[3]);
    const int K = static_cast<int>(k.shape()[0]), R = static_cast<int>(k.shape()[2]), S = static_cast<int>(k.shape()[3]);
    ck(sdb_conv_dgrad(context(), dt_code(x.dtype()), ddy.p, dkin.p, ddx.p, N, H, W, C, K, R, S, stride, pad, 0,
                      nullptr));
    ck(sdb_conv_wgrad(context(), dt_code(x.dtype()), dxin.p, ddy.p, ddk.p, N, H, W, C, K, R, S, stride, pad,
                      nullptr));
    return {download_nchw(ddx, s, x.dtype(), DType::F32), download_nchw(ddk, k.shape(), x.dtype(), DType::F32)};
}

std::pair<Tensor, BNStats> syncbn_forward(const Tensor& x, std::span<const float> gamma,
                                          std::span<const float> beta, float eps, CommGroup* group) {
    check_nchw(x, "syncbn_forward");
    if (group && group->size() > 1)
        throw ContractError("simdet::gpu::syncbn_forward: cross-GPU groups are libsdb contexts (sdb_syncbn_fwd)");
    const int64_t C = x.shape()[1], rows = x.shape()[0] * x.shape()[2] * x.shape()[3];
    if (static_cast<int64_t>(gamma.size()) != C || static_cast<int64_t>(beta.size()) != C)
        throw ShapeError("syncbn_forward: gamma/beta length differs from the channel count");
    Dev dx(dev_bytes(x)), dy(dev_bytes(x)), dg(C * 4), db(C * 4), mu(C * 4), is(C * 4), agg((2 * C + 1) * 4);
    upload_nhwc(x, dx);
    upload_vec(gamma, dg);
    upload_vec(beta, db);
    // the world-1 group path returns the reference's 2C+1 float aggregation buffer
    ck(sdb_syncbn_fwd(context(), dt_code(x.dtype()), dx.p, dg.f(), db.f(), dy.p, mu.f(), is.f(), agg.f(), rows,
                      static_cast<int>(C), eps, 0, nullptr));
    BNStats st;
    const auto a = download_vec(agg, static_cast<size_t>(2 * C + 1));
    st.sum.assign(a.begin(), a.begin() + C);
    st.sumsq.assign(a.begin() + C, a.begin() + 2 * C);
    st.count = static_cast<int64_t>(a[2 * C]);
    st.mean = download_vec(mu, static_cast<size_t>(C));
    st.invstd = download_vec(is, static_cast<size_t>(C));
    return {download_nchw(dy, x.shape(), x.dtype(), x.dtype()), std::move(st)};
}

BnGrads syncbn_backward(const Tensor& dy_in, const Tensor& x, const BNStats& stats, std::span<const float> gamma,
                        CommGroup* group) {
    check_nchw(x, "syncbn_backward");
    if (group && group->size() > 1)
        throw ContractError("simdet::gpu::syncbn_backward: cross-GPU groups are libsdb contexts (sdb_syncbn_bwd)");
    const Tensor dy = dy_in.astype(x.dtype());
    const int64_t C = x.shape()[1], rows = x.shape()[0] * x.shape()[2] * x.shape()[3];
    if (static_cast<int64_t>(stats.mean.size()) != C || static_cast<int64_t>(stats.invstd.size()) != C)
        throw ContractError("syncbn_backward: statistics do not match the input");
    Dev dx(dev_bytes(x)), ddy(dev_bytes(x)), ddx(dev_bytes(x)), dg(C * 4), mu(C * 4), is(C * 4), ogm(C * 4), obt(C * 4);
    upload_nhwc(x, dx);
    upload_nhwc(dy, ddy);
    upload_vec(gamma, dg);
    upload_vec(stats.mean, mu);
    upload_vec(stats.invstd, is);
    ck(sdb_bn_bwd(context(), dt_code(x.dtype()), ddy.p, dx.p, nullptr, dg.f(), mu.f(), is.f(), ddx.p, ogm.f(), obt.f(),
                  rows, static_cast<int>(C), nullptr));
    BnGrads g;
    g.dx = download_nchw(ddx, x.shape(), x.dtype(), DType::F32);
    g.dgamma = download_vec(ogm, static_cast<size_t>(C));
    g.dbeta = download_vec(obt, static_cast<size_t>(C));
    return g;
}

std::pair<Tensor, IabnSaved> iabn_forward(const Tensor& x, std::span<const float> gamma, std::span<const float> beta,
                                          float eps, float slope) {
    check_nchw(x, "iabn_forward");
    const int64_t C = x.shape()[1], rows = x.shape()[0] * x.shape()[2] * x.shape()[3];
    if (static_cast<int64_t>(gamma.size()) != C || static_cast<int64_t>(beta.size()) != C)
        throw ShapeError("iabn_forward: gamma/beta length differs from the channel count");
    Dev dx(dev_bytes(x)), dy(dev_bytes(x)), dg(C * 4), db(C * 4), mu(C * 4), is(C * 4);
    upload_nhwc(x, dx);
    upload_vec(gamma, dg);
    upload_vec(beta, db);
    ck(sdb_iabn_fwd(context(), dt_code(x.dtype()), dx.p, dg.f(), db.f(), dy.p, mu.f(), is.f(), rows,
                    static_cast<int>(C), eps, slope, nullptr));
    IabnSaved sv;
    sv.y = download_nchw(dy, x.shape(), x.dtype(), x.dtype());
    sv.mean = download_vec(mu, static_cast<size_t>(C));
    sv.invstd = download_vec(is, static_cast<size_t>(C));
    sv.gamma.assign(gamma.begin(), gamma.end());
    sv.beta.assign(beta.begin(), beta.end());
    sv.eps = eps;
    sv.slope = slope;
    Tensor y = sv.y;
    return {std::move(y), std::move(sv)};
}

IabnGrads iabn_backward(const Tensor& dy_in, const IabnSaved& sv) {
    check_nchw(sv.y, "iabn_backward");
    const Tensor dy = dy_in.astype(sv.y.dtype());
    const int64_t C = sv.y.shape()[1], rows = sv.y.shape()[0] * sv.y.shape()[2] * sv.y.shape()[3];
    Dev dyy(dev_bytes(sv.y)), ddy(dev_bytes(sv.y)), ddx(dev_bytes(sv.y)), dg(C * 4), db(C * 4), mu(C * 4), is(C * 4),
        ogm(C * 4), obt(C * 4);
    upload_nhwc(sv.y, dyy);
    upload_nhwc(dy, ddy);
    upload_vec(sv.gamma, dg);
    upload_vec(sv.beta, db);
    upload_vec(sv.mean, mu);
    upload_vec(sv.invstd, is);
    ck(sdb_iabn_bwd(context(), dt_code(sv.y.dtype()), ddy.p, dyy.p, dg.f(), db.f(), mu.f(), is.f(), ddx.p, ogm.f(),
                    obt.f(), rows, static_cast<int>(C), sv.slope, nullptr));
    IabnGrads g;
    g.dx = download_nchw(ddx, sv.y.shape(), sv.y.dtype(), DType::F32);
    g.dgamma = download_vec(ogm, static_cast<size_t>(C));
    g.dbeta = download_vec(obt, static_cast<size_t>(C));
    return g;
}

bool apply_sgd(std::span<float> w, std::span<float> v, std::span<const float> gsum, float lr, float momentum,
               double scale, int K) {
    if (w.size() != v.size() || w.size() != gsum.size()) throw ContractError("apply_sgd: length mismatch");
    const size_t n = w.size();
    Dev dw(n * 4), dv(n * 4), dg(n * 4), dflag(4), dscale(8);
    upload_vec(w, dw);
    upload_vec(v, dv);
    upload_vec(gsum, dg);
    const int zero = 0;
    ck(sdb_copy_to_device(context(), dflag.p, &zero, 4));
    ck(sdb_copy_to_device(context(), dscale.p, &scale, 8));
    ck(sdb_nonfinite(context(), SDB_F32, dg.p, static_cast<int64_t>(n), static_cast<int*>(dflag.p), nullptr));
    ck(sdb_fused_sgd(context(), SDB_F32, dg.p, dw.f(), dv.f(), nullptr, static_cast<int64_t>(n), lr, momentum,
                     static_cast<const double*>(dscale.p), static_cast<double>(K), static_cast<const int*>(dflag.p),
                     nullptr));
    int flag = 0;
    ck(sdb_copy_to_host(context(), &flag, dflag.p, 4));
    if (flag) return true;  // overflow: w and v untouched (trainer.cpp:253)
    ck(sdb_copy_to_host(context(), w.data(), dw.p, n * 4));
    ck(sdb_copy_to_host(context(), v.data(), dv.p, n * 4));
    return false;
}

}  // namespace simdet::gpu
