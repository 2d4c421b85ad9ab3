// norm.cu -- BatchNorm and InPlace-ABN forward/backward on NHWC tensors.
//
// Reference semantics (all under /root/reference/proj/src):
//   BN fwd   syncbn.cpp:21-70  FP64 per-channel sum/sumsq, sums rounded to
//            float (agg buffer), mean = sum/count, biased var clamped >= 0,
//            invstd = 1/sqrt(var+eps), y = gamma*(x-mean)*invstd + beta.
//   BN bwd   syncbn.cpp:72-117 FP64 sum(dy), sum(dy*xhat) (rounded to float),
//            dx = gamma*invstd*(dy - s1/m - xhat*s2/m), dgamma = s2, dbeta = s1.
//   IABN fwd memopt.cpp:226-276 same statistics kept in double, y = leaky(z).
//   IABN bwd memopt.cpp:278-327 recompute z and xhat from the OUTPUT y
//            (z = y>=0 ? y : y/slope; xhat = (z-beta)/gamma), dz = dy*(y>0?1:slope).
// The optional fused ReLU of the BN path (C1: BN followed by relu,
// model.cpp:238-245) keeps its mask in the stored output (y>0 <=> z>0).
//
// Kernels: (1) per-block partial statistics: a producer lane streams 16 KB
// row tiles into a shared-memory ring with cp.async.bulk, 8 consumer warps
// (8 channels per thread) accumulate every element in fp64 exactly like the
// reference, fp64 block reduction -> partial[block][2C]; (2) fixed-order fp64
// finalize per channel (deterministic, no atomics); (3) apply through the same
// bulk-copy ring, float expressions evaluated in the reference's order
// without FMA contraction.  The second read of x in (3) mostly hits the
// 126 MB L2.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "sdb_internal.h"

namespace sdb {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxBlocks = 2 * kNumSMs;

template <class T>
SDB_DEV void load8(const T* p, float (&v)[8]);
template <>
SDB_DEV void load8<__half>(const __half* p, float (&v)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __half22float2(h[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
    }
}
template <>
SDB_DEV void load8<float>(const float* p, float (&v)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
// Packed fp32 pairs (sm_100 add/mul.rn.f32x2): each lane is exactly the scalar
// round-to-nearest operation, so the IABN expressions below stay bit-identical
// to their scalar forms (a - b is issued as a + (-b), x * k2 subtracted as
// x * (-k2): both exact sign identities) at half the FP32 instruction count.
// ptxas (12.9) contracts a packed multiply feeding a packed add into FFMA2
// (one rounding instead of two) even for explicit mul.rn/add.rn.f32x2 PTX and
// -fmad=false; a packed product feeding SCALAR add.rn stays two roundings.
// So: add2 only where no product feeds it, add2s (two scalar adds) after a
// product.
SDB_DEV float2 mul2(float2 a, float2 b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;"
        : "=l"(r)
        : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
    return *reinterpret_cast<const float2*>(&r);
}
SDB_DEV float2 add2(float2 a, float2 b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(r)
        : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
    return *reinterpret_cast<const float2*>(&r);
}
SDB_DEV float2 add2s(float2 a, float2 b) { return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y)); }
SDB_DEV float2 pair(const float (&v)[8], int j) { return make_float2(v[j], v[j + 1]); }

// InPlace-ABN backward for channels j, j+1 of one row (memopt.cpp:278-327):
// z = y >= 0 ? y : y / slope (as y * (1/slope)), dz = dy * (y > 0 ? 1 : slope),
// xhat = (z - beta) * (1/gamma)
SDB_DEV void iabn_bwd_pair(const float (&y)[8], const float (&dy)[8], int j, float2 inv_slope2, float slope,
                           float2 nbeta, float2 igamma, float2& dz, float2& xh) {
    const float2 ys = mul2(pair(y, j), inv_slope2);
    const float2 z = make_float2(y[j] >= 0.f ? y[j] : ys.x, y[j + 1] >= 0.f ? y[j + 1] : ys.y);
    dz = mul2(pair(dy, j), make_float2(y[j] > 0.f ? 1.f : slope, y[j + 1] > 0.f ? 1.f : slope));
    xh = mul2(add2(z, nbeta), igamma);
}

template <class T>
SDB_DEV void store8(T* p, const float (&v)[8]);
template <>
SDB_DEV void store8<__half>(__half* p, const float (&v)[8]) {
    uint4 u;
    __half2* h = reinterpret_cast<__half2*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = u;
}
template <>
SDB_DEV void store8<float>(float* p, const float (&v)[8]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}

// ---------------------------------------------------------------- statistics
// KIND 0: (x, x^2)             forward statistics
// KIND 1: (dz, dz*xhat) BN     xhat = (x-mean)*invstd (float), dz = relu mask ? dy : 0
// KIND 2: (dz, dz*xhat) IABN   recompute from y
struct StatArgs {
    const void* a;  // x (KIND 0/1) or y (KIND 2)
    const void* dy;
    const void* y;  // BN relu mask source (may be null)
    const float *gamma, *beta, *mean, *invstd;
    float slope;
    int64_t rows;
    int C;
    int64_t rows_per_block;
    double* partial;
    int keep_l2;  // operands small enough to stay in L2 for the apply pass
    // KIND 4: dy is the average-pool backward of pooled [rows / pool_hw][C],
    // masked by the sign bitmap in the `dy` slot (C / 8 bytes per row):
    // dy = rn(bit ? rn(g * inv) : neg * rn(g * inv)) exactly as avgpool_bwd
    // stores it, which this pass also writes to dy_out
    const void* pooled;
    float pool_inv, pool_neg;
    int pool_hw;
    void* dy_out;
};

// the masked average-pool gradient of one row's 8 channels (avgpool_bwd's
// arithmetic); the scaled pooled values are cached per pooling group (a
// thread walks consecutive rows, 49 per RoI)
// Row -> (group, index in group) without a 64-bit division per row: the
// callers (C / 8 == threads, one thread per 8 channels) visit every row of
// their range in order, so the position advances by one per call.
struct GroupPos {
    int64_t grp = -1;
    int ig = 0;
    SDB_DEV void next(int64_t row, int hw) {
        if (grp < 0) {
            grp = row / hw;
            ig = static_cast<int>(row - grp * hw);
        } else if (++ig == hw) {
            ig = 0;
            ++grp;
        }
    }
};
struct PooledCache {
    GroupPos pos;
    int64_t loaded = -1;
    float r[8];
};
template <class T>
SDB_DEV void pooled_dy8(const T* pooled, int64_t row, int pool_hw, int C, int c0, float inv, float neg,
                        unsigned int bm, PooledCache& pc, float (&d)[8]) {
    pc.pos.next(row, pool_hw);
    if (pc.pos.grp != pc.loaded) {
        float g[8];
        load8<T>(pooled + pc.pos.grp * C + c0, g);
#pragma unroll
        for (int j = 0; j < 8; ++j) pc.r[j] = to_f<T>(from_f<T>(g[j] * inv));
        pc.loaded = pc.pos.grp;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = to_f<T>(from_f<T>(((bm >> j) & 1u) ? pc.r[j] : neg * pc.r[j]));
}

// Bulk-copy pipeline: a producer lane streams contiguous row tiles (16 KB per
// operand) into a ring of shared-memory stages with cp.async.bulk (completion
// by transaction bytes on an mbarrier); 8 consumer warps reduce each tile from
// shared memory.  Memory-level parallelism is ST x NIN x 16 KB per CTA
// (~96 KB), independent of registers, which is what keeps HBM busy: the
// previous register-pipelined version sat at 25% occupancy and ~2.7 TB/s.
constexpr int kTileBytes = 16384;
constexpr int kStatThreads = kThreads + 32;  // + producer warp

template <int NIN>
struct StatPipe {
    static constexpr int kStages = NIN == 1 ? 6 : (NIN == 2 ? 3 : 2);
    static constexpr int kSmem = kStages * NIN * kTileBytes + 2 * kStages * 8;
};

// rows per tile for channel count C
template <class T>
SDB_DEV int tile_rows_for(int C) {
    return kTileBytes / (C * static_cast<int>(sizeof(T)));
}

// producer lane: stream row tiles [r_begin, r_end) of up to three operands
// into the stage ring
// hint: 0 default, 1 evict_last (a second pass follows), 2 evict_first (last read)
// rowb1 > 0: operand 1 has rowb1 bytes per row (a sign bitmap) instead of C x T
template <class T, int NIN, int ST>
SDB_DEV void stream_tiles(uint32_t sbase, uint64_t* full, uint64_t* empty, const void* a, const void* b,
                          const void* c, int64_t r_begin, int64_t r_end, int ntiles, int TR, int C, int hint = 0,
                          int rowb1 = 0) {
    const uint8_t* src[3] = {static_cast<const uint8_t*>(a), static_cast<const uint8_t*>(b),
                             static_cast<const uint8_t*>(c)};
    const int64_t rb = static_cast<int64_t>(C) * sizeof(T);
    const uint64_t pol = hint == 1 ? l2_evict_last_policy() : (hint == 2 ? l2_evict_first_policy() : 0ull);
    for (int i = 0; i < ntiles; ++i) {
        const int s = i % ST;
        if (i >= ST) mbar_wait(&empty[s], ((i / ST) - 1) & 1);
        const int64_t r0 = r_begin + static_cast<int64_t>(i) * TR;
        const int nr = static_cast<int>(min(static_cast<int64_t>(TR), r_end - r0));
        const uint32_t bytes = static_cast<uint32_t>(nr * rb);
        const uint32_t bytes1 = rowb1 ? static_cast<uint32_t>(nr) * rowb1 : bytes;
        mbar_arrive_expect_tx(&full[s], bytes * NIN + (NIN > 1 ? bytes1 - bytes : 0u));
#pragma unroll
        for (int j = 0; j < NIN; ++j) {
            const int64_t rbj = (j == 1 && rowb1) ? rowb1 : rb;
            const uint32_t by = j == 1 ? bytes1 : bytes;
            if (hint) bulk_load_hint(sbase + (s * NIN + j) * kTileBytes, src[j] + r0 * rbj, by, &full[s], pol);
            else bulk_load(sbase + (s * NIN + j) * kTileBytes, src[j] + r0 * rbj, by, &full[s]);
        }
    }
}

template <class T, int KIND, int NIN>
__global__ void __launch_bounds__(kStatThreads, 2) stats_kernel(StatArgs p) {
    constexpr int ST = StatPipe<NIN>::kStages;
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + ST * NIN * kTileBytes);
    uint64_t* empty = full + ST;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int C = p.C;
    const int TR = tile_rows_for<T>(C);
    const int64_t r_begin = blockIdx.x * p.rows_per_block;
    const int64_t r_end = min(p.rows, r_begin + p.rows_per_block);
    const int ntiles = r_end > r_begin ? static_cast<int>((r_end - r_begin + TR - 1) / TR) : 0;
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kThreads / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();
    pdl_wait();
    pdl_trigger();
    const uint32_t sbase = smem_u32(sm);
    const int tpr = C / 8;
    const int rpi = kThreads / tpr;
    const int cg = tid % tpr, rg = tid / tpr;
    const int c0 = cg * 8;
    double S[8], Q[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) S[j] = Q[j] = 0.0;
    if (warp == kThreads / 32) {
        // ------------------------------------------------ producer
        if (lane == 0)
            stream_tiles<T, NIN, ST>(sbase, full, empty, p.a, p.dy, p.y, r_begin, r_end, ntiles, TR, C,
                                     p.keep_l2 ? 1 : 0, KIND == 4 ? C / 8 : 0);
    } else {
        // ------------------------------------------------ consumers
        float g[8], b[8], mu[8], is[8];
        if (KIND != 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                g[j] = p.gamma[c0 + j];
                is[j] = p.invstd[c0 + j];
                mu[j] = KIND == 1 ? p.mean[c0 + j] : 0.f;
                b[j] = KIND >= 2 ? -p.beta[c0 + j] : 0.f;  // negated: z + (-beta)
                if (KIND >= 2) g[j] = 1.0f / g[j];          // xhat = (z - beta) * (1/gamma)
            }
        }
        const float inv_slope = 1.0f / p.slope;
        const float2 inv_slope2 = make_float2(inv_slope, inv_slope);
        PooledCache pcache;  // KIND 4
        // Every element is accumulated in fp64 exactly as the reference does
        // (syncbn.cpp:29-39, memopt.cpp:250-258 / 305-314): the float value
        // widened to double, the product formed exactly in double (fma of two
        // widened floats rounds once, like `s += (double)a * b`).  Only the
        // order of the fp64 additions differs, so the float-rounded sums, and
        // with them mean/invstd, agree with the reference to the last bit
        // almost always.
        for (int i = 0; i < ntiles; ++i) {
            const int st = i % ST;
            mbar_wait(&full[st], (i / ST) & 1);
            const int64_t r0 = r_begin + static_cast<int64_t>(i) * TR;
            const int nr = static_cast<int>(min(static_cast<int64_t>(TR), r_end - r0));
            const T* ta = reinterpret_cast<const T*>(sm + (st * NIN) * kTileBytes);
            const T* td = reinterpret_cast<const T*>(sm + (st * NIN + 1) * kTileBytes);
            const T* tm = reinterpret_cast<const T*>(sm + (st * NIN + 2) * kTileBytes);
            for (int rr = rg; rr < nr; rr += rpi) {
                const int off = rr * C + c0;
                float v[8], dd[8], ym[8];
                load8<T>(ta + off, v);
                if (KIND == 4) {
                    const unsigned int bm = reinterpret_cast<const uint8_t*>(td)[rr * (C / 8) + cg];
                    pooled_dy8<T>(static_cast<const T*>(p.pooled), r0 + rr, p.pool_hw, C, c0, p.pool_inv,
                                  p.pool_neg, bm, pcache, dd);
                    store8<T>(static_cast<T*>(p.dy_out) + (r0 + rr) * C + c0, dd);
                } else if (KIND != 0) {
                    load8<T>(td + off, dd);
                }
                if (NIN == 3) load8<T>(tm + off, ym);
                if (KIND == 0) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const double dv = static_cast<double>(v[j]);
                        S[j] = __dadd_rn(S[j], dv);
                        Q[j] = __fma_rn(dv, dv, Q[j]);
                    }
                } else if (KIND == 1) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float d = (NIN == 3 && !(ym[j] > 0.f)) ? 0.f : dd[j];
                        const float xh = __fmul_rn(__fsub_rn(v[j], mu[j]), is[j]);
                        S[j] = __dadd_rn(S[j], static_cast<double>(d));
                        Q[j] = __fma_rn(static_cast<double>(d), static_cast<double>(xh), Q[j]);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 8; j += 2) {
                        float2 dz, xh;
                        iabn_bwd_pair(v, dd, j, inv_slope2, p.slope, pair(b, j), pair(g, j), dz, xh);
                        S[j] = __dadd_rn(S[j], static_cast<double>(dz.x));
                        Q[j] = __fma_rn(static_cast<double>(dz.x), static_cast<double>(xh.x), Q[j]);
                        S[j + 1] = __dadd_rn(S[j + 1], static_cast<double>(dz.y));
                        Q[j + 1] = __fma_rn(static_cast<double>(dz.y), static_cast<double>(xh.y), Q[j + 1]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
    }
    // every stage has been consumed (all bulk copies landed): reuse the ring
    // as the fixed-order block reduction buffer, laid out [value][thread] so a
    // warp's stores and loads hit consecutive banks
    __syncthreads();
    double* red = reinterpret_cast<double*>(sm);
    if (tid < kThreads && rg != 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            red[j * kThreads + tid] = S[j];
            red[(8 + j) * kThreads + tid] = Q[j];
        }
    }
    __syncthreads();
    if (tid < kThreads && rg == 0) {
        for (int k = 1; k < rpi; ++k) {
            const int t = k * tpr + cg;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                S[j] += red[j * kThreads + t];
                Q[j] += red[(8 + j) * kThreads + t];
            }
        }
        double* out = p.partial + static_cast<int64_t>(blockIdx.x) * 2 * C;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            out[c0 + j] = S[j];
            out[C + c0 + j] = Q[j];
        }
    }
}

// MODE 0: BN fwd (sums rounded to float first), 1: IABN fwd (double)
// MODE 2: BN bwd, 3: IABN bwd  -> coef[0..C) = s1/m, coef[C..2C) = s2/m
// MODE 4/5: SyncBN fwd/bwd local sums as floats into coef (+ count for 4)
// Fixed-order parallel reduction of the per-block partials, spread over many
// SMs (8 channels per CTA): thread (ch, g) of 128 groups loads partial[b][c] for
// b = g, g+128, g+256 in one L2 round trip and adds them in block order; the
// 128 group sums are combined by a fixed tree (shuffles inside a warp, then the
// 32 warp sums through shared memory).  Deterministic, no atomics.
constexpr int kFinCh = 8;
constexpr int kFinThreads = 1024;
constexpr int kFinGroups = kFinThreads / kFinCh;
__global__ void __launch_bounds__(kFinThreads) finalize_kernel(const double* __restrict__ partial, int nblocks, int C,
                                                               int64_t count, float eps, int mode, float* mean,
                                                               float* invstd, float* dgamma, float* dbeta,
                                                               float* coef) {
    __shared__ double rs[32][kFinCh], rq[32][kFinCh];
    pdl_wait();
    pdl_trigger();
    const int ch = threadIdx.x % kFinCh, g = threadIdx.x / kFinCh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * kFinCh + ch;
    // -0.0 is the exact additive identity (keeps the sign of an all -0 sum)
    double S = -0.0, Q = -0.0;
    if (c < C) {
        const int64_t stride = 2 * static_cast<int64_t>(C);
        constexpr int kPer = (kMaxBlocks + kFinGroups - 1) / kFinGroups;
        double sv[kPer], qv[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int b = g + kFinGroups * u;
            sv[u] = b < nblocks ? partial[b * stride + c] : -0.0;
            qv[u] = b < nblocks ? partial[b * stride + C + c] : -0.0;
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            S += sv[u];
            Q += qv[u];
        }
    }
    // groups 4w..4w+3 of warp w: fixed pairwise tree
#pragma unroll
    for (int o = kFinCh; o < 32; o <<= 1) {
        S += __shfl_xor_sync(0xffffffffu, S, o);
        Q += __shfl_xor_sync(0xffffffffu, Q, o);
    }
    if (lane < kFinCh) {
        rs[warp][lane] = S;
        rq[warp][lane] = Q;
    }
    __syncthreads();
    if (warp != 0) return;
    // lane = (ch, quarter): 4 quarters of 8 warp sums each, then a 2-level tree
    const int qtr = lane / kFinCh;
    S = -0.0;
    Q = -0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        S += rs[qtr * 8 + k][ch];
        Q += rq[qtr * 8 + k][ch];
    }
#pragma unroll
    for (int o = kFinCh; o < 32; o <<= 1) {
        S += __shfl_xor_sync(0xffffffffu, S, o);
        Q += __shfl_xor_sync(0xffffffffu, Q, o);
    }
    if (lane >= kFinCh || c >= C) return;
    if (mode == 4 || mode == 5) {
        // SyncBN: this rank's sums rounded to float into the reduction buffer
        // [S_0..S_{C-1}, Q_0..Q_{C-1}(, count)] (src/syncbn.cpp:27-40 / 83-95)
        coef[c] = static_cast<float>(S);
        coef[C + c] = static_cast<float>(Q);
        if (mode == 4 && c == 0) coef[2 * C] = static_cast<float>(count);
        return;
    }
    if (mode == 0 || mode == 1) {
        double mu, var;
        if (mode == 0) {
            const float sf = static_cast<float>(S), qf = static_cast<float>(Q);
            mu = static_cast<double>(sf) / static_cast<double>(count);
            var = static_cast<double>(qf) / static_cast<double>(count) - mu * mu;
        } else {
            mu = S / static_cast<double>(count);
            var = Q / static_cast<double>(count) - mu * mu;
        }
        if (var < 0.0) var = 0.0;
        mean[c] = static_cast<float>(mu);
        invstd[c] = static_cast<float>(1.0 / sqrt(var + static_cast<double>(eps)));
    } else {
        const float s1 = static_cast<float>(S), s2 = static_cast<float>(Q);
        dgamma[c] = s2;
        dbeta[c] = s1;
        if (mode == 2) {
            const float m = static_cast<float>(count);
            coef[c] = s1 / m;
            coef[C + c] = s2 / m;
        } else {
            coef[c] = static_cast<float>(S / static_cast<double>(count));
            coef[C + c] = static_cast<float>(Q / static_cast<double>(count));
        }
    }
}

// ---------------------------------------------------------------- apply
// KIND 0: BN fwd (+act relu when act==1), 1: IABN fwd, 2: BN bwd, 3: IABN bwd,
// 4: IABN fwd + residual add + act, 6: 4 + average pool (out2 not stored)
struct ApplyArgs {
    const void* a;   // x or y
    const void* dy;
    const void* y;   // relu mask (BN bwd)
    void* out;
    const float *gamma, *beta, *mean, *invstd, *coef;
    float slope;
    int act;
    int64_t n8;  // number of 8-element groups
    int C;
    // KIND 4 (IABN fwd fused with the residual add + activation): the shortcut
    // arrives through the `dy` slot, out2 = act2(round(y) + shortcut)
    void* out2;
    int act2;
    float slope2;
    // optional sign bitmap of the stored out2 (bit j of byte [row][c/8] = out2 > 0),
    // what the dgrad epilogue of the next layer needs of it
    uint8_t* bits;
    // KIND 6 (KIND 4 closing the RoI head, C/8 == kThreads): out2 is not
    // stored; its rows are average-pooled per group of pool_hw rows into
    // pooled [rows / pool_hw][C] (fp32 sums in row order, / pool_hw, rounded:
    // avgpool_fwd's arithmetic) and only its sign bitmap is kept
    void* pooled;
    int pool_hw;
    // KIND 7 (IABN bwd, dy = the masked average-pool gradient as in KIND 4 of
    // the statistics pass; the sign bitmap streams in the `dy` slot)
    float pool_inv, pool_neg;
};

SDB_DEV void ldf8(const float* p, float (&v)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// Same bulk-copy pipeline as the statistics pass: the producer lane streams
// the operand row tiles into shared memory, the 8 consumer warps (one 8-channel
// group per thread, parameters in registers) normalise from shared memory and
// store 128-bit rows straight to HBM.  Safe in place (out == a or out == dy):
// a tile is read into shared memory before any of its rows is written, and
// only this CTA touches its rows.
template <class T, int KIND, int NIN>
__global__ void __launch_bounds__(kStatThreads, 2) apply_kernel(ApplyArgs p, int64_t rows, int64_t rpb) {
    constexpr int ST = StatPipe<NIN>::kStages;
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + ST * NIN * kTileBytes);
    uint64_t* empty = full + ST;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int C = p.C;
    const int TR = tile_rows_for<T>(C);
    const int64_t r_begin = blockIdx.x * rpb;
    const int64_t r_end = min(rows, r_begin + rpb);
    const int ntiles = r_end > r_begin ? static_cast<int>((r_end - r_begin + TR - 1) / TR) : 0;
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kThreads / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();
    pdl_wait();
    pdl_trigger();
    if (warp == kThreads / 32) {
        if (lane == 0)
            stream_tiles<T, NIN, ST>(smem_u32(sm), full, empty, p.a, p.dy, p.y, r_begin, r_end, ntiles, TR, C, 2,
                                     KIND == 7 ? C / 8 : 0);
        return;
    }
    const int tpr = C / 8;
    const int rpi = kThreads / tpr;
    const int cg = tid % tpr, rg = tid / tpr;
    const int c0 = cg * 8;
    float g[8], b[8], mu[8], is[8], k1[8], k2[8];
    ldf8(p.gamma + c0, g);
    ldf8(p.invstd + c0, is);
    if (KIND != 3 && KIND != 7) ldf8(p.mean + c0, mu);
    if (KIND != 2) ldf8(p.beta + c0, b);
    if (KIND >= 2) {
        ldf8(p.coef + c0, k1);
        ldf8(p.coef + C + c0, k2);
    }
    float ig[8], gis[8], nmu[8], nb[8], nk1[8], nk2[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        ig[j] = 1.0f / g[j];
        gis[j] = __fmul_rn(g[j], is[j]);
        nmu[j] = KIND != 3 && KIND != 7 ? -mu[j] : 0.f;
        nb[j] = KIND != 2 ? -b[j] : 0.f;
        nk1[j] = KIND >= 2 ? -k1[j] : 0.f;
        nk2[j] = KIND >= 2 ? -k2[j] : 0.f;
    }
    const float inv_slope = 1.0f / p.slope;
    const float2 inv_slope2 = make_float2(inv_slope, inv_slope);
    const float2 slope2 = make_float2(p.slope, p.slope);
    T* out = static_cast<T*>(p.out);
    float pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // KIND 6: this thread's channels, rows in order
    PooledCache pcache;                        // KIND 7
    GroupPos ppos;                             // KIND 6
    for (int i = 0; i < ntiles; ++i) {
        const int st = i % ST;
        mbar_wait(&full[st], (i / ST) & 1);
        const int64_t r0 = r_begin + static_cast<int64_t>(i) * TR;
        const int nr = static_cast<int>(min(static_cast<int64_t>(TR), r_end - r0));
        const T* ta = reinterpret_cast<const T*>(sm + (st * NIN) * kTileBytes);
        const T* td = reinterpret_cast<const T*>(sm + (st * NIN + 1) * kTileBytes);
        const T* tm = reinterpret_cast<const T*>(sm + (st * NIN + 2) * kTileBytes);
        for (int rr = rg; rr < nr; rr += rpi) {
            const int off = rr * C + c0;
            float v[8], o[8];
            load8<T>(ta + off, v);
            if (KIND == 0 || KIND == 1 || KIND == 4 || KIND == 6) {
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    // gamma*(x-mean)*invstd + beta, evaluated like the reference (no contraction)
                    const float2 z =
                        add2s(mul2(mul2(pair(g, j), add2(pair(v, j), pair(nmu, j))), pair(is, j)), pair(b, j));
                    if (KIND == 0) {
                        o[j] = (p.act && !(z.x > 0.f)) ? 0.f : z.x;
                        o[j + 1] = (p.act && !(z.y > 0.f)) ? 0.f : z.y;
                    } else {
                        const float2 zs = mul2(slope2, z);
                        o[j] = z.x > 0.f ? z.x : zs.x;
                        o[j + 1] = z.y > 0.f ? z.y : zs.y;
                    }
                }
                if (KIND == 4 || KIND == 6) {
                    // residual node: s = round(round(y) + shortcut) (src/tensor.cpp:125), then
                    // relu / leaky, exactly as the separate add_act pass
                    float sc[8], o2[8];
                    load8<T>(td + off, sc);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float yr = to_f<T>(from_f<T>(o[j]));
                        const float sr = to_f<T>(from_f<T>(__fadd_rn(yr, sc[j])));
                        o2[j] = p.act2 == 0 ? sr : (sr > 0.f ? sr : (p.act2 == 1 ? 0.f : __fmul_rn(p.slope2, sr)));
                    }
                    if (KIND == 4) {
                        store8<T>(static_cast<T*>(p.out2) + (r0 + rr) * C + c0, o2);
                    } else {
                        // rpi == 1: this thread sees every row of its pooling groups in order
                        ppos.next(r0 + rr, p.pool_hw);
                        const int64_t grp = ppos.grp;
                        const int ig = ppos.ig;
#pragma unroll
                        for (int j = 0; j < 8; ++j) pacc[j] = (ig == 0 ? 0.f : pacc[j]) + to_f<T>(from_f<T>(o2[j]));
                        if (ig == p.pool_hw - 1) {
                            float pm[8];
#pragma unroll
                            for (int j = 0; j < 8; ++j) pm[j] = pacc[j] / static_cast<float>(p.pool_hw);
                            store8<T>(static_cast<T*>(p.pooled) + grp * C + c0, pm);
                        }
                    }
                    if (p.bits) {
                        uint32_t bm = 0;
#pragma unroll
                        for (int j = 0; j < 8; ++j) bm |= (to_f<T>(from_f<T>(o2[j])) > 0.f ? 1u : 0u) << j;
                        p.bits[(r0 + rr) * (C / 8) + cg] = static_cast<uint8_t>(bm);
                    }
                }
            } else {
                float d[8];
                if (KIND == 7) {
                    const unsigned int bm = reinterpret_cast<const uint8_t*>(td)[rr * (C / 8) + cg];
                    pooled_dy8<T>(static_cast<const T*>(p.pooled), r0 + rr, p.pool_hw, C, c0, p.pool_inv, p.pool_neg,
                                  bm, pcache, d);
                } else {
                    load8<T>(td + off, d);
                }
                if (KIND == 2) {
                    if (NIN == 3) {
                        float yv[8];
                        load8<T>(tm + off, yv);
#pragma unroll
                        for (int j = 0; j < 8; ++j) d[j] = yv[j] > 0.f ? d[j] : 0.f;
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        // gis * (dy - s1 - xh * s2), syncbn.cpp:110-111 (no contraction)
                        const float xh = __fmul_rn(__fsub_rn(v[j], mu[j]), is[j]);
                        o[j] = __fmul_rn(gis[j], __fsub_rn(__fsub_rn(d[j], k1[j]), __fmul_rn(xh, k2[j])));
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 8; j += 2) {
                        // gis * ((dz - s1) - xh * s2) (memopt.cpp:318-322), no contraction
                        float2 dz, xh;
                        iabn_bwd_pair(v, d, j, inv_slope2, p.slope, pair(nb, j), pair(ig, j), dz, xh);
                        const float2 r =
                            mul2(pair(gis, j), add2s(add2s(dz, pair(nk1, j)), mul2(xh, pair(nk2, j))));
                        o[j] = r.x;
                        o[j + 1] = r.y;
                    }
                }
            }
            store8<T>(out + (r0 + rr) * C + c0, o);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
}

// SyncBN statistics from the (all-reduced) float buffer agg = [sum, sumsq,
// count] -- src/syncbn.cpp:43-57 -- and backward coefficients from red =
// [sum dy, sum dy*xhat] with the forward's global count (src/syncbn.cpp:98-111)
__global__ void syncbn_stats_kernel(const float* __restrict__ agg, int C, float eps, float* __restrict__ mean,
                                    float* __restrict__ invstd) {
    pdl_wait();
    pdl_trigger();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    const int64_t count = static_cast<int64_t>(agg[2 * C]);
    const double mu = static_cast<double>(agg[c]) / static_cast<double>(count);
    double var = static_cast<double>(agg[C + c]) / static_cast<double>(count) - mu * mu;
    if (var < 0.0) var = 0.0;
    mean[c] = static_cast<float>(mu);
    invstd[c] = static_cast<float>(1.0 / sqrt(var + static_cast<double>(eps)));
}

__global__ void syncbn_coef_kernel(const float* __restrict__ red, const float* __restrict__ agg_fwd, int C,
                                   float* __restrict__ dgamma, float* __restrict__ dbeta, float* __restrict__ coef) {
    pdl_wait();
    pdl_trigger();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    const float m = static_cast<float>(static_cast<int64_t>(agg_fwd[2 * C]));
    const float s1 = red[c], s2 = red[C + c];
    dgamma[c] = s2;
    dbeta[c] = s1;
    coef[c] = s1 / m;
    coef[C + c] = s2 / m;
}

// Finalize from an fprop's fused statistics (ConvStats): channel c lives in
// n-tile nt = c / bn at column j = c % bn of the CTAs b = nt, nt + tiles_n, ...
// (T = 4 * ctas / tiles_n quadrant terms).  Same thread layout and fixed
// reduction tree as finalize_kernel (8 channels per CTA, 128 term groups).
constexpr int kConvTermsMax = 2 * kNumSMs * 4;
// mode 0 / 1: BN / IABN forward statistics -> mean, invstd; mode 3: IABN
// backward sums from a dgrad epilogue -> dgamma, dbeta, coef (as finalize_kernel)
__global__ void __launch_bounds__(kFinThreads) finalize_conv_kernel(const double* __restrict__ cs, int ctas, int tiles_n,
                                                                    int bn, int C, int64_t count, float eps, int mode,
                                                                    float* mean, float* invstd, float* dgamma = nullptr,
                                                                    float* dbeta = nullptr, float* coef = nullptr) {
    __shared__ double rs[32][kFinCh], rq[32][kFinCh];
    pdl_wait();
    pdl_trigger();
    const int ch = threadIdx.x % kFinCh, g = threadIdx.x / kFinCh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * kFinCh + ch;
    double S = -0.0, Q = -0.0;
    if (c < C) {
        const int nt = c / bn, j = c - nt * bn;
        const int T = 4 * (ctas / tiles_n);
        constexpr int kPer = (kConvTermsMax + kFinGroups - 1) / kFinGroups;
        double sv[kPer], qv[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int t = g + kFinGroups * u;
            if (t < T) {
                const int b = nt + (t >> 2) * tiles_n, q = t & 3;
                const double* p = cs + (static_cast<int64_t>(b) * 4 + q) * 2 * bn + j;
                sv[u] = p[0];
                qv[u] = p[bn];
            } else {
                sv[u] = -0.0;
                qv[u] = -0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            S += sv[u];
            Q += qv[u];
        }
    }
#pragma unroll
    for (int o = kFinCh; o < 32; o <<= 1) {
        S += __shfl_xor_sync(0xffffffffu, S, o);
        Q += __shfl_xor_sync(0xffffffffu, Q, o);
    }
    if (lane < kFinCh) {
        rs[warp][lane] = S;
        rq[warp][lane] = Q;
    }
    __syncthreads();
    if (warp != 0) return;
    const int qtr = lane / kFinCh;
    S = -0.0;
    Q = -0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        S += rs[qtr * 8 + k][ch];
        Q += rq[qtr * 8 + k][ch];
    }
#pragma unroll
    for (int o = kFinCh; o < 32; o <<= 1) {
        S += __shfl_xor_sync(0xffffffffu, S, o);
        Q += __shfl_xor_sync(0xffffffffu, Q, o);
    }
    if (lane >= kFinCh || c >= C) return;
    if (mode == 3) {
        dgamma[c] = static_cast<float>(Q);
        dbeta[c] = static_cast<float>(S);
        coef[c] = static_cast<float>(S / static_cast<double>(count));
        coef[C + c] = static_cast<float>(Q / static_cast<double>(count));
        return;
    }
    double mu, var;
    if (mode == 0) {
        const float sf = static_cast<float>(S), qf = static_cast<float>(Q);
        mu = static_cast<double>(sf) / static_cast<double>(count);
        var = static_cast<double>(qf) / static_cast<double>(count) - mu * mu;
    } else {
        mu = S / static_cast<double>(count);
        var = Q / static_cast<double>(count) - mu * mu;
    }
    if (var < 0.0) var = 0.0;
    mean[c] = static_cast<float>(mu);
    invstd[c] = static_cast<float>(1.0 / sqrt(var + static_cast<double>(eps)));
}

struct Plan {
    int nblocks;
    int64_t rpb;
};

// Rows are split into at most 2 CTAs per SM, each a whole number of tiles.
Plan plan_for(int64_t rows, int C, int elem_bytes) {
    const int64_t tr = kTileBytes / (static_cast<int64_t>(C) * elem_bytes);
    const int64_t tiles = std::max<int64_t>(1, (rows + tr - 1) / tr);
    const int64_t nb = std::min<int64_t>(tiles, kMaxBlocks);
    const int64_t tpb = (tiles + nb - 1) / nb;
    Plan p;
    p.rpb = tpb * tr;
    p.nblocks = static_cast<int>((rows + p.rpb - 1) / p.rpb);
    if (p.nblocks < 1) p.nblocks = 1;
    return p;
}

template <class T, int KIND, int NIN>
cudaError_t run_stats(const StatArgs& a0, const Plan& pl, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(stats_kernel<T, KIND, NIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             StatPipe<NIN>::kSmem);
        configured = true;
    }
    StatArgs a = a0;
    a.rows_per_block = pl.rpb;
    // the apply pass re-reads the same operands: keep them in L2 when they fit
    // in well under half of its 126 MB
    a.keep_l2 = static_cast<double>(a.rows) * a.C * sizeof(T) * NIN <= 48e6 ? 1 : 0;
    return launch_pdl(stats_kernel<T, KIND, NIN>, dim3(pl.nblocks), dim3(kStatThreads), StatPipe<NIN>::kSmem, st, a);
}

template <class T, int KIND, int NIN>
cudaError_t run_apply(const ApplyArgs& aa, int64_t rows, const Plan& pl, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(apply_kernel<T, KIND, NIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             StatPipe<NIN>::kSmem);
        configured = true;
    }
    return launch_pdl(apply_kernel<T, KIND, NIN>, dim3(pl.nblocks), dim3(kStatThreads), StatPipe<NIN>::kSmem, st, aa,
                      rows, pl.rpb);
}

void finalize(const double* partial, const Plan& pl, int C, int64_t rows, float eps, int mode, float* mean,
              float* invstd, float* dgamma, float* dbeta, float* coef, cudaStream_t st) {
    launch_pdl(finalize_kernel, dim3((C + kFinCh - 1) / kFinCh), dim3(kFinThreads), 0, st, partial, pl.nblocks, C, rows, eps, mode, mean,
               invstd, dgamma, dbeta, coef);
}

}  // namespace

bool norm_channels_ok(int C) { return C >= 8 && C <= 2048 && (C % 8) == 0 && (2048 % C) == 0; }

size_t norm_workspace_bytes(int64_t rows, int C) {
    // the fp16 plan has the most blocks (fewest rows per tile)... take the max of both
    const Plan p16 = plan_for(std::max<int64_t>(rows, 1), C, 2);
    const Plan p32 = plan_for(std::max<int64_t>(rows, 1), C, 4);
    const int nb = std::max(p16.nblocks, p32.nblocks);
    return static_cast<size_t>(nb) * 2 * C * sizeof(double) + 2 * C * sizeof(float) + 256;
}

cudaError_t bn_forward(int dtype, const void* x, const float* gamma, const float* beta, void* y, float* mean,
                       float* invstd, int64_t rows, int C, float eps, int act, float slope, void* ws, cudaStream_t st) {
    // act: 0 none, 1 relu (BN mode);  act 2 = IABN with `slope`
    const Plan pl = plan_for(rows, C, dtype == kF16 ? 2 : 4);
    double* partial = static_cast<double*>(ws);
    StatArgs sa{};
    sa.a = x; sa.rows = rows; sa.C = C; sa.partial = partial; sa.slope = 1.f;
    cudaError_t e = dtype == kF16 ? run_stats<__half, 0, 1>(sa, pl, st) : run_stats<float, 0, 1>(sa, pl, st);
    if (e != cudaSuccess) return e;
    finalize(partial, pl, C, rows, eps, act == 2 ? 1 : 0, mean, invstd, nullptr, nullptr, nullptr, st);
    ApplyArgs aa{};
    aa.a = x; aa.out = y; aa.gamma = gamma; aa.beta = beta; aa.mean = mean; aa.invstd = invstd;
    aa.slope = slope; aa.act = act; aa.n8 = rows * C / 8; aa.C = C;
    if (act == 2) return dtype == kF16 ? run_apply<__half, 1, 1>(aa, rows, pl, st) : run_apply<float, 1, 1>(aa, rows, pl, st);
    return dtype == kF16 ? run_apply<__half, 0, 1>(aa, rows, pl, st) : run_apply<float, 0, 1>(aa, rows, pl, st);
}

cudaError_t bn_forward_stats(int dtype, const void* x, float* mean, float* invstd, int64_t rows, int C, float eps,
                             int act, void* ws, cudaStream_t st) {
    const Plan pl = plan_for(rows, C, dtype == kF16 ? 2 : 4);
    double* partial = static_cast<double*>(ws);
    StatArgs sa{};
    sa.a = x; sa.rows = rows; sa.C = C; sa.partial = partial; sa.slope = 1.f;
    cudaError_t e = dtype == kF16 ? run_stats<__half, 0, 1>(sa, pl, st) : run_stats<float, 0, 1>(sa, pl, st);
    if (e != cudaSuccess) return e;
    finalize(partial, pl, C, rows, eps, act == 2 ? 1 : 0, mean, invstd, nullptr, nullptr, nullptr, st);
    return cudaGetLastError();
}

cudaError_t bn_apply_add_act(int dtype, const void* x, const float* gamma, const float* beta, const float* mean,
                             const float* invstd, void* y, const void* shortcut, void* out, int64_t rows, int C,
                             float slope, int act2, float slope2, cudaStream_t st, uint8_t* out_bits) {
    const Plan pl = plan_for(rows, C, dtype == kF16 ? 2 : 4);
    ApplyArgs aa{};
    aa.bits = out_bits;
    aa.a = x; aa.dy = shortcut; aa.out = y; aa.gamma = gamma; aa.beta = beta; aa.mean = mean; aa.invstd = invstd;
    aa.slope = slope; aa.act = 2; aa.n8 = rows * C / 8; aa.C = C;
    aa.out2 = out; aa.act2 = act2; aa.slope2 = slope2;
    return dtype == kF16 ? run_apply<__half, 4, 2>(aa, rows, pl, st) : run_apply<float, 4, 2>(aa, rows, pl, st);
}

cudaError_t bn_apply_add_act_pool(int dtype, const void* x, const float* gamma, const float* beta, const float* mean,
                                  const float* invstd, void* y, const void* shortcut, void* pooled, int pool_hw,
                                  int64_t rows, int C, float slope, int act2, float slope2, cudaStream_t st,
                                  uint8_t* out_bits) {
    const int eb = dtype == kF16 ? 2 : 4;
    if (C / 8 != kThreads || pool_hw < 1 || rows % pool_hw != 0 || !out_bits) return cudaErrorInvalidValue;
    // one pooling group (RoI) per CTA, its last tile partial: 1024 CTAs at C4
    // balance better than whole-tile multiples of the group (warm ncu: 138 us
    // vs 149-150 us with 2 or 4 groups per CTA)
    (void)eb;
    Plan pl;
    pl.rpb = pool_hw;
    pl.nblocks = static_cast<int>((rows + pl.rpb - 1) / pl.rpb);
    ApplyArgs aa{};
    aa.bits = out_bits;
    aa.a = x; aa.dy = shortcut; aa.out = y; aa.gamma = gamma; aa.beta = beta; aa.mean = mean; aa.invstd = invstd;
    aa.slope = slope; aa.act = 2; aa.n8 = rows * C / 8; aa.C = C;
    aa.act2 = act2; aa.slope2 = slope2; aa.pooled = pooled; aa.pool_hw = pool_hw;
    return dtype == kF16 ? run_apply<__half, 6, 2>(aa, rows, pl, st) : run_apply<float, 6, 2>(aa, rows, pl, st);
}

cudaError_t iabn_backward_pooled(int dtype, const void* pooled, const uint8_t* bits, int pool_hw, float neg,
                                 const void* y, const float* gamma, const float* beta, const float* invstd,
                                 void* dy_out, void* dx, float* dgamma, float* dbeta, int64_t rows, int C, float slope,
                                 void* ws, cudaStream_t st) {
    if (C / 8 != kThreads || pool_hw < 1 || rows % pool_hw != 0) return cudaErrorInvalidValue;
    const Plan pl = plan_for(rows, C, dtype == kF16 ? 2 : 4);
    double* partial = static_cast<double*>(ws);
    float* coef = reinterpret_cast<float*>(partial + static_cast<int64_t>(pl.nblocks) * 2 * C);
    const float inv = static_cast<float>(1.0 / static_cast<double>(pool_hw));  // as avgpool_bwd
    StatArgs sa{};
    sa.a = y; sa.dy = bits; sa.gamma = gamma; sa.beta = beta; sa.invstd = invstd; sa.slope = slope;
    sa.rows = rows; sa.C = C; sa.partial = partial;
    sa.pooled = pooled; sa.pool_inv = inv; sa.pool_neg = neg; sa.pool_hw = pool_hw; sa.dy_out = dy_out;
    cudaError_t e = dtype == kF16 ? run_stats<__half, 4, 2>(sa, pl, st) : run_stats<float, 4, 2>(sa, pl, st);
    if (e != cudaSuccess) return e;
    finalize(partial, pl, C, rows, 0.f, 3, nullptr, nullptr, dgamma, dbeta, coef, st);
    ApplyArgs aa{};
    aa.a = y; aa.dy = bits; aa.out = dx; aa.gamma = gamma; aa.beta = beta; aa.invstd = invstd; aa.coef = coef;
    aa.slope = slope; aa.n8 = rows * C / 8; aa.C = C;
    aa.pooled = const_cast<void*>(pooled); aa.pool_hw = pool_hw; aa.pool_inv = inv; aa.pool_neg = neg;
    return dtype == kF16 ? run_apply<__half, 7, 2>(aa, rows, pl, st) : run_apply<float, 7, 2>(aa, rows, pl, st);
}

cudaError_t bn_backward(int dtype, const void* dy, const void* x, const void* y_mask, const float* gamma,
                        const float* mean, const float* invstd, void* dx, float* dgamma, float* dbeta, int64_t rows,
                        int C, void* ws, cudaStream_t st) {
    const Plan pl = plan_for(rows, C, dtype == kF16 ? 2 : 4);
    double* partial = static_cast<double*>(ws);
    float* coef = reinterpret_cast<float*>(partial + static_cast<int64_t>(pl.nblocks) * 2 * C);
    StatArgs sa{};
    sa.a = x; sa.dy = dy; sa.y = y_mask; sa.gamma = gamma; sa.mean = mean; sa.invstd = invstd;
    sa.rows = rows; sa.C = C; sa.partial = partial; sa.slope = 1.f;
    cudaError_t e;
    if (y_mask) e = dtype == kF16 ? run_stats<__half, 1, 3>(sa, pl, st) : run_stats<float, 1, 3>(sa, pl, st);
    else e = dtype == kF16 ? run_stats<__half, 1, 2>(sa, pl, st) : run_stats<float, 1, 2>(sa, pl, st);
    if (e != cudaSuccess) return e;
    finalize(partial, pl, C, rows, 0.f, 2, nullptr, nullptr, dgamma, dbeta, coef, st);
    ApplyArgs aa{};
    aa.a = x; aa.dy = dy; aa.y = y_mask; aa.out = dx; aa.gamma = gamma; aa.mean = mean; aa.invstd = invstd;
    aa.coef = coef; aa.n8 = rows * C / 8; aa.C = C;
    if (y_mask)
        return dtype == kF16 ? run_apply<__half, 2, 3>(aa, rows, pl, st) : run_apply<float, 2, 3>(aa, rows, pl, st);
    return dtype == kF16 ? run_apply<__half, 2, 2>(aa, rows, pl, st) : run_apply<float, 2, 2>(aa, rows, pl, st);
}

cudaError_t iabn_backward(int dtype, const void* dy, const void* y, const float* gamma, const float* beta,
                          const float* mean, const float* invstd, void* dx, float* dgamma, float* dbeta, int64_t rows,
                          int C, float slope, void* ws, cudaStream_t st) {
    (void)mean;
    const Plan pl = plan_for(rows, C, dtype == kF16 ? 2 : 4);
    double* partial = static_cast<double*>(ws);
    float* coef = reinterpret_cast<float*>(partial + static_cast<int64_t>(pl.nblocks) * 2 * C);
    StatArgs sa{};
    sa.a = y; sa.dy = dy; sa.gamma = gamma; sa.beta = beta; sa.invstd = invstd; sa.slope = slope;
    sa.rows = rows; sa.C = C; sa.partial = partial;
    cudaError_t e = dtype == kF16 ? run_stats<__half, 2, 2>(sa, pl, st) : run_stats<float, 2, 2>(sa, pl, st);
    if (e != cudaSuccess) return e;
    finalize(partial, pl, C, rows, 0.f, 3, nullptr, nullptr, dgamma, dbeta, coef, st);
    ApplyArgs aa{};
    aa.a = y; aa.dy = dy; aa.out = dx; aa.gamma = gamma; aa.beta = beta; aa.invstd = invstd; aa.coef = coef;
    aa.slope = slope; aa.n8 = rows * C / 8; aa.C = C;
    return dtype == kF16 ? run_apply<__half, 3, 2>(aa, rows, pl, st) : run_apply<float, 3, 2>(aa, rows, pl, st);
}

// ---------------------------------------------------------------- fused statistics
// mean/invstd from an fprop's fused output statistics (act == 2: IABN double
// statistics, else BN float-rounded sums), then (y != nullptr) the apply pass
cudaError_t bn_forward_conv_stats(int dtype, const void* x, const float* gamma, const float* beta, void* y,
                                  float* mean, float* invstd, int64_t rows, int C, float eps, int act, float slope,
                                  const ConvStats& cs, cudaStream_t st) {
    if (!cs.produced || 4 * (cs.ctas / cs.tiles_n) > kConvTermsMax) return cudaErrorInvalidValue;
    cudaError_t e = launch_pdl(finalize_conv_kernel, dim3((C + kFinCh - 1) / kFinCh), dim3(kFinThreads), 0, st, cs.buf,
                               cs.ctas, cs.tiles_n, cs.bn, C, rows, eps, act == 2 ? 1 : 0, mean, invstd,
                               static_cast<float*>(nullptr), static_cast<float*>(nullptr), static_cast<float*>(nullptr));
    if (e != cudaSuccess || !y) return e;
    const Plan pl = plan_for(rows, C, dtype == kF16 ? 2 : 4);
    ApplyArgs aa{};
    aa.a = x; aa.out = y; aa.gamma = gamma; aa.beta = beta; aa.mean = mean; aa.invstd = invstd;
    aa.slope = slope; aa.act = act; aa.n8 = rows * C / 8; aa.C = C;
    if (act == 2) return dtype == kF16 ? run_apply<__half, 1, 1>(aa, rows, pl, st) : run_apply<float, 1, 1>(aa, rows, pl, st);
    return dtype == kF16 ? run_apply<__half, 0, 1>(aa, rows, pl, st) : run_apply<float, 0, 1>(aa, rows, pl, st);
}

cudaError_t iabn_backward_conv_stats(int dtype, const void* dy, const void* y, const float* gamma, const float* beta,
                                     const float* invstd, void* dx, float* dgamma, float* dbeta, int64_t rows, int C,
                                     float slope, const ConvStats& cs, float* coef, cudaStream_t st) {
    if (!cs.produced || 4 * (cs.ctas / cs.tiles_n) > kConvTermsMax) return cudaErrorInvalidValue;
    cudaError_t e = launch_pdl(finalize_conv_kernel, dim3((C + kFinCh - 1) / kFinCh), dim3(kFinThreads), 0, st, cs.buf,
                               cs.ctas, cs.tiles_n, cs.bn, C, rows, 0.f, 3, static_cast<float*>(nullptr),
                               static_cast<float*>(nullptr), dgamma, dbeta, coef);
    if (e != cudaSuccess) return e;
    const Plan pl = plan_for(rows, C, dtype == kF16 ? 2 : 4);
    ApplyArgs aa{};
    aa.a = y; aa.dy = dy; aa.out = dx; aa.gamma = gamma; aa.beta = beta; aa.invstd = invstd; aa.coef = coef;
    aa.slope = slope; aa.n8 = rows * C / 8; aa.C = C;
    return dtype == kF16 ? run_apply<__half, 3, 2>(aa, rows, pl, st) : run_apply<float, 3, 2>(aa, rows, pl, st);
}

// ---------------------------------------------------------------- SyncBN
cudaError_t syncbn_local_sums(int dtype, const void* x, int64_t rows, int C, float* agg, void* ws, cudaStream_t st) {
    const Plan pl = plan_for(rows, C, dtype == kF16 ? 2 : 4);
    double* partial = static_cast<double*>(ws);
    StatArgs sa{};
    sa.a = x; sa.rows = rows; sa.C = C; sa.partial = partial; sa.slope = 1.f;
    cudaError_t e = dtype == kF16 ? run_stats<__half, 0, 1>(sa, pl, st) : run_stats<float, 0, 1>(sa, pl, st);
    if (e != cudaSuccess) return e;
    finalize(partial, pl, C, rows, 0.f, 4, nullptr, nullptr, nullptr, nullptr, agg, st);
    return cudaGetLastError();
}

cudaError_t syncbn_forward_finish(int dtype, const void* x, const float* gamma, const float* beta, void* y,
                                  float* mean, float* invstd, const float* agg, int64_t rows, int C, float eps,
                                  int act, cudaStream_t st) {
    cudaError_t e = launch_pdl(syncbn_stats_kernel, dim3((C + 255) / 256), dim3(256), 0, st, agg, C, eps, mean, invstd);
    if (e != cudaSuccess) return e;
    const Plan pl = plan_for(rows, C, dtype == kF16 ? 2 : 4);
    ApplyArgs aa{};
    aa.a = x; aa.out = y; aa.gamma = gamma; aa.beta = beta; aa.mean = mean; aa.invstd = invstd;
    aa.slope = 1.f; aa.act = act; aa.n8 = rows * C / 8; aa.C = C;
    return dtype == kF16 ? run_apply<__half, 0, 1>(aa, rows, pl, st) : run_apply<float, 0, 1>(aa, rows, pl, st);
}

cudaError_t syncbn_backward_local_sums(int dtype, const void* dy, const void* x, const void* y_mask,
                                       const float* mean, const float* invstd, float* red, int64_t rows, int C,
                                       void* ws, cudaStream_t st) {
    const Plan pl = plan_for(rows, C, dtype == kF16 ? 2 : 4);
    double* partial = static_cast<double*>(ws);
    StatArgs sa{};
    sa.a = x; sa.dy = dy; sa.y = y_mask; sa.mean = mean; sa.invstd = invstd;
    sa.rows = rows; sa.C = C; sa.partial = partial; sa.slope = 1.f;
    cudaError_t e;
    if (y_mask) e = dtype == kF16 ? run_stats<__half, 1, 3>(sa, pl, st) : run_stats<float, 1, 3>(sa, pl, st);
    else e = dtype == kF16 ? run_stats<__half, 1, 2>(sa, pl, st) : run_stats<float, 1, 2>(sa, pl, st);
    if (e != cudaSuccess) return e;
    finalize(partial, pl, C, rows, 0.f, 5, nullptr, nullptr, nullptr, nullptr, red, st);
    return cudaGetLastError();
}

cudaError_t syncbn_backward_finish(int dtype, const void* dy, const void* x, const void* y_mask, const float* gamma,
                                   const float* mean, const float* invstd, const float* red, const float* agg_fwd,
                                   void* dx, float* dgamma, float* dbeta, int64_t rows, int C, void* ws,
                                   cudaStream_t st) {
    float* coef = static_cast<float*>(ws);
    cudaError_t e = launch_pdl(syncbn_coef_kernel, dim3((C + 255) / 256), dim3(256), 0, st, red, agg_fwd, C, dgamma,
                               dbeta, coef);
    if (e != cudaSuccess) return e;
    const Plan pl = plan_for(rows, C, dtype == kF16 ? 2 : 4);
    ApplyArgs aa{};
    aa.a = x; aa.dy = dy; aa.y = y_mask; aa.out = dx; aa.gamma = gamma; aa.mean = mean; aa.invstd = invstd;
    aa.coef = coef; aa.n8 = rows * C / 8; aa.C = C;
    if (y_mask)
        return dtype == kF16 ? run_apply<__half, 2, 3>(aa, rows, pl, st) : run_apply<float, 2, 3>(aa, rows, pl, st);
    return dtype == kF16 ? run_apply<__half, 2, 2>(aa, rows, pl, st) : run_apply<float, 2, 2>(aa, rows, pl, st);
}

}  // namespace sdb
