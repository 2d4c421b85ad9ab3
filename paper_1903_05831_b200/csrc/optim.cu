// optim.cu -- the loss-scaled mixed-precision update (north-star item 4).
//
// Restates, bit for bit, the reference's step tail (src/trainer.cpp):
//   has_nonfinite(gsum)                       trainer.cpp:78-82, used at :252
//   apply_sgd: inv = float(1/(scale*K)); g = gsum*inv; v = mu*v + g;
//              w -= lr*v   (all FP32)           trainer.cpp:86-94, used at :253-254
//   fp16 shadow refresh of conv/fc weights     trainer.cpp:222-227
//   update_scale(ls, overflow)                 precision.cpp:45-56, used at :257
// Every float operation is an explicit _rn intrinsic so no FMA contraction
// can change the bits.  The loss scale lives in device memory (no host sync
// on the overflow flag); the update is skipped on device when the flag is set.
#include <algorithm>

#include "common.cuh"
#include "sdb_internal.h"

namespace sdb {

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n, int per_thread) {
    const int64_t b = (n + static_cast<int64_t>(kThreads) * per_thread - 1) / (static_cast<int64_t>(kThreads) * per_thread);
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, 8 * kNumSMs)));
}

template <class T>
__global__ void nonfinite_kernel(const T* __restrict__ g, int64_t n, int* __restrict__ flag) {
    int bad = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float v = to_f<T>(g[i]);
        bad |= !isfinite(v);
    }
    bad = __syncthreads_or(bad);
    if (bad && threadIdx.x == 0) atomicOr(flag, 1);
}

// vectorised fp16 variant: 8 halves per 16-byte load
__global__ void nonfinite_h8_kernel(const uint4* __restrict__ g, int64_t n8, int* __restrict__ flag) {
    int bad = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint4 u = g[i];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            // a binary16 is non-finite iff its exponent field is all ones
            bad |= ((w[k] & 0x7c00u) == 0x7c00u) | (((w[k] >> 16) & 0x7c00u) == 0x7c00u);
        }
    }
    bad = __syncthreads_or(bad);
    if (bad && threadIdx.x == 0) atomicOr(flag, 1);
}

template <class T>
__global__ void fused_sgd_kernel(const T* __restrict__ gsum, float* __restrict__ w, float* __restrict__ v,
                                 __half* __restrict__ w16, int64_t n, float lr, float mu, const double* __restrict__ scale,
                                 double denom_mult, const int* __restrict__ flag) {
    if (flag && *flag) return;  // overflow: weights and velocity untouched (trainer.cpp:253)
    const double denom = __dmul_rn(scale ? *scale : 1.0, denom_mult);
    const float inv = __double2float_rn(__ddiv_rn(1.0, denom));
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float g = __fmul_rn(to_f<T>(gsum[i]), inv);
        const float vi = __fadd_rn(__fmul_rn(mu, v[i]), g);
        const float wi = __fsub_rn(w[i], __fmul_rn(lr, vi));
        v[i] = vi;
        w[i] = wi;
        if (w16) w16[i] = __float2half_rn(wi);
    }
}

// fp16 gradients, 8 parameters per thread per iteration: 16-byte loads of g
// and of the fp16 shadow, 32-byte loads/stores of w and v (n % 8 == 0, all
// pointers 16-byte aligned); per element the same _rn expression as above
__global__ void __launch_bounds__(256) fused_sgd_h8_kernel(const uint4* __restrict__ gsum, float4* __restrict__ w,
                                                           float4* __restrict__ v, uint4* __restrict__ w16, int64_t n8,
                                                           float lr, float mu, const double* __restrict__ scale,
                                                           double denom_mult, const int* __restrict__ flag) {
    if (flag && *flag) return;  // overflow: weights and velocity untouched (trainer.cpp:253)
    const double denom = __dmul_rn(scale ? *scale : 1.0, denom_mult);
    const float inv = __double2float_rn(__ddiv_rn(1.0, denom));
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint4 gu = gsum[i];
        const __half2* g2 = reinterpret_cast<const __half2*>(&gu);
        float4 wa = w[2 * i], wb = w[2 * i + 1], va = v[2 * i], vb = v[2 * i + 1];
        float* wf[8] = {&wa.x, &wa.y, &wa.z, &wa.w, &wb.x, &wb.y, &wb.z, &wb.w};
        float* vf[8] = {&va.x, &va.y, &va.z, &va.w, &vb.x, &vb.y, &vb.z, &vb.w};
        uint4 hu;
        __half2* h2 = reinterpret_cast<__half2*>(&hu);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 gf = __half22float2(g2[k]);
            float o[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int e = 2 * k + q;
                const float g = __fmul_rn(q ? gf.y : gf.x, inv);
                const float vi = __fadd_rn(__fmul_rn(mu, *vf[e]), g);
                const float wi = __fsub_rn(*wf[e], __fmul_rn(lr, vi));
                *vf[e] = vi;
                *wf[e] = wi;
                o[q] = wi;
            }
            h2[k] = __floats2half2_rn(o[0], o[1]);
        }
        w[2 * i] = wa;
        w[2 * i + 1] = wb;
        v[2 * i] = va;
        v[2 * i + 1] = vb;
        if (w16) w16[i] = hu;
    }
}

__global__ void update_scale_kernel(double* scale, int64_t* good, const int* flag, int dynamic, int64_t interval,
                                    double growth, double backoff, double min_scale, double max_scale) {
    if (!dynamic) return;
    if (*flag) {
        *scale = fmax(min_scale, __dmul_rn(*scale, backoff));
        *good = 0;
        return;
    }
    if (++*good >= interval) {
        *scale = fmin(max_scale, __dmul_rn(*scale, growth));
        *good = 0;
    }
}

__global__ void cast_f32_f16_kernel(const float* __restrict__ in, __half* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __float2half_rn(in[i]);
}
__global__ void cast_f16_f32_kernel(const __half* __restrict__ in, float* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __half2float(in[i]);
}

}  // namespace

cudaError_t nonfinite_check(int gdtype, const void* g, int64_t n, int* flag, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (gdtype == kF16 && (reinterpret_cast<uintptr_t>(g) & 15) == 0 && (n & 7) == 0) {
        nonfinite_h8_kernel<<<grid_for(n / 8, 4), kThreads, 0, st>>>(static_cast<const uint4*>(g), n / 8, flag);
    } else if (gdtype == kF16) {
        nonfinite_kernel<__half><<<grid_for(n, 8), kThreads, 0, st>>>(static_cast<const __half*>(g), n, flag);
    } else {
        nonfinite_kernel<float><<<grid_for(n, 8), kThreads, 0, st>>>(static_cast<const float*>(g), n, flag);
    }
    return cudaGetLastError();
}

cudaError_t fused_sgd(int gdtype, const void* gsum, float* w, float* v, __half* w16, int64_t n, float lr, float mu,
                      const double* scale, double denom_mult, const int* flag, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (gdtype == kF16 && (n & 7) == 0 && al16(gsum) && al16(w) && al16(v) && (!w16 || al16(w16))) {
        fused_sgd_h8_kernel<<<grid_for(n / 8, 2), kThreads, 0, st>>>(
            static_cast<const uint4*>(gsum), reinterpret_cast<float4*>(w), reinterpret_cast<float4*>(v),
            reinterpret_cast<uint4*>(w16), n / 8, lr, mu, scale, denom_mult, flag);
    } else if (gdtype == kF16)
        fused_sgd_kernel<__half><<<grid_for(n, 4), kThreads, 0, st>>>(static_cast<const __half*>(gsum), w, v, w16, n, lr,
                                                                     mu, scale, denom_mult, flag);
    else
        fused_sgd_kernel<float><<<grid_for(n, 4), kThreads, 0, st>>>(static_cast<const float*>(gsum), w, v, w16, n, lr,
                                                                    mu, scale, denom_mult, flag);
    return cudaGetLastError();
}

cudaError_t update_scale_device(double* scale, int64_t* good, const int* flag, int dynamic, int64_t interval,
                                double growth, double backoff, double min_scale, double max_scale, cudaStream_t st) {
    update_scale_kernel<<<1, 1, 0, st>>>(scale, good, flag, dynamic, interval, growth, backoff, min_scale, max_scale);
    return cudaGetLastError();
}

cudaError_t cast_f32_f16(const float* in, __half* out, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    cast_f32_f16_kernel<<<grid_for(n, 4), kThreads, 0, st>>>(in, out, n);
    return cudaGetLastError();
}
cudaError_t cast_f16_f32(const __half* in, float* out, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    cast_f16_f32_kernel<<<grid_for(n, 4), kThreads, 0, st>>>(in, out, n);
    return cudaGetLastError();
}

}  // namespace sdb
