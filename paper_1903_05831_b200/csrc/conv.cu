// conv.cu -- convolution (reference K1/K2: src/tensor.cpp:157-196 forward,
// src/autograd.cpp:290-320 backward) as implicit GEMM on the sm_100a tensor
// cores (tcgen05.mma kind::f16, fp32 accumulators in TMEM).
//
// Layouts: activations NHWC, filters KRSC ([out][kh][kw][in]), fp16 storage,
// fp32 accumulation, outputs rounded RNE (the reference's fp16 contract,
// src/tensor.cpp:79-82 + 195).
//
//   fprop : Y[m=(n,oh,ow)][k]     = sum_{(r,s,c)} X[n,oh*st-p+r,ow*st-p+s,c] * W[k,r,s,c]
//   dgrad : DX[m=(n,h,w)][c]      = sum_{(r,s,k)} DY[n,(h+p-r)/st,(w+p-s)/st,k] * W[k,r,s,c]
//           (sub-pixel phases: each stride phase (h%st,w%st) is its own GEMM over
//            the taps that land on it, so stride-2 layers waste no MACs)
//   wgrad : DW[k][(r,s,c)]        = sum_{m=(n,oh,ow)} DY[m][k] * X[n,oh*st-p+r,ow*st-p+s,c]
//           (deterministic split-K over m: fp32 partials reduced in fixed order)
//
// Mainloop: 4 producer warps gather the implicit-im2col tiles with 16-byte
// cp.async (zero-fill gives the padding) straight into the UMMA SWIZZLE_128B
// canonical layouts (K-major or MN-major, so no transposes are ever
// materialised), completion is published through mbarriers after a
// fence.proxy.async; one elected thread issues tcgen05.mma into TMEM and
// releases stages with tcgen05.commit; the same 4 warps then drain TMEM with
// tcgen05.ld and write the epilogue.  A CUDA-core variant of the same GEMM
// views serves fp32 mode (config C1: reference-precision) and odd channel
// counts.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include <cuda.h>

#include "common.cuh"
#include "sdb_internal.h"

namespace sdb {

bool pdl_enabled() {
    static const bool e = std::getenv("SDB_NO_PDL") == nullptr;
    return e;
}

enum ConvMode { FPROP = 0, DGRAD = 1, WGRAD = 2 };

struct ConvArgs {
    const void* x;   // fprop/wgrad: input activation; dgrad: DY
    const void* w;   // fprop/dgrad: filter; wgrad: DY
    void* out;       // fprop: Y, dgrad: DX, wgrad: DW or fp32 partials
    int N, H, W, C, K, R, S, stride, pad, Ho, Wo;
    int M, NG, KG;   // GEMM extents
    // dgrad phase
    int ph, pw, Hp, Wp, r0, nr, q0, nq;
    // wgrad split-K
    int kb_per_split;
    int accumulate;  // dgrad: out = result + addend
    const void* addend;  // dgrad accumulate source (may alias out)
    // dgrad: gradient through the activation that produced the layer input:
    // out = round(round(result + addend) * (mask > 0 ? 1 : mask_neg)) -- the
    // separate act_bwd pass (src/autograd.cpp:340-351) folded into the epilogue
    const void* mask;
    float mask_neg;
    int tma_b;       // dgrad: filter operand loaded by TMA (needs K % 64 == 0)
    int plain;       // 1x1 / stride 1 / pad 0: the activation operand is a plain 2-D [pixels][channels] tile
    int tma_out;     // fp16 output written by TMA stores from swizzled staging (tm.o)
    const uint8_t* mbits;  // dgrad: sign bitmap of the mask tensor (bit c%8 of byte [row][c/8] = mask > 0)
    // fprop with the TMA-store epilogue: per-channel FP64 [sum, sumsq] of the
    // rounded fp16 output, accumulated by each CTA over its tiles (one n-tile
    // per CTA) and written as stats[cta][quadrant][2][BN] (norm statistics fused)
    double* stats;
    // dgrad EPI 2: the InPlace-ABN backward statistics of the layer whose output
    // gradient this dgrad produces (src/memopt.cpp:305-314): per column c,
    // [sum dz | sum dz*xhat] with dz = dy*(y > 0 ? 1 : slope), xhat = (z - beta)/gamma,
    // z = y >= 0 ? y : y/slope; y is read by TMA alongside the output tile
    const float* bs_gamma;
    const float* bs_beta;
    float bs_slope;
};

// TMA descriptors of the dense GEMM operand (filter for fprop/dgrad, DY for wgrad)
struct alignas(64) TmaDesc {
    CUtensorMap m;
};

// ============================================================ tcgen05 kernel
constexpr int kBM = 128, kBK = 64;

// byte offset of 16B chunk inside a K-major SW128 tile: (row, chunk of 8 k)
SDB_DEV uint32_t kmaj_off(int row, int chunk) {
    return static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 128 + (((chunk ^ row) & 7) << 4));
}
// byte offset of 16B chunk inside an MN-major SW128 tile of MN extent E:
// (mn chunk index mc = mn/8, k row)
SDB_DEV uint32_t mnmaj_off(int mc, int k, int E) {
    return static_cast<uint32_t>((k >> 3) * (E / 64) * 1024 + (mc >> 3) * 1024 + (k & 7) * 128 +
                                 (((mc ^ k) & 7) << 4));
}

// Epilogue of one output tile, run by the 4 epilogue warps (warp w owns TMEM
// lane quadrant q = w & 3, i.e. tile rows 32q..32q+31): TMEM -> registers
// (16 columns at a time) -> XOR-swizzled smem staging -> coalesced 16-byte
// stores (fp16 RNE, fp32 split-K partials for wgrad, optional dgrad addend).
// The accumulator is handed back to the MMA warp as soon as it is drained.
template <int MODE, int BN>
SDB_DEV void epilogue_tile(const ConvArgs& a, int split, int m0, int n0, int nk, uint32_t tacc, int q, int lane,
                           float* stg, uint64_t* tempty_acc) {
    // row pointers of the 2 rows each lane stores in the coalesced phase
    int64_t rowp[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int r = (k * 32 + lane) >> 1;  // 0..31
        const int grow = m0 + q * 32 + r;
        int64_t o = -1;
        if (grow < a.M) {
            if (MODE == FPROP) {
                o = static_cast<int64_t>(grow) * a.NG;
            } else if (MODE == DGRAD) {
                const int HpWp = a.Hp * a.Wp;
                const int n = grow / HpWp, rem = grow - n * HpWp, i2 = rem / a.Wp, j2 = rem - i2 * a.Wp;
                o = ((static_cast<int64_t>(n) * a.H + a.ph + a.stride * i2) * a.W + a.pw + a.stride * j2) * a.C;
            } else {
                o = (static_cast<int64_t>(split) * a.M + grow) * a.NG;
            }
        }
        rowp[k] = o;
    }
    const int lim = MODE == DGRAD ? a.C : a.NG;
#pragma unroll 1
    for (int cb = 0; cb < BN; cb += 16) {
        // residual fan-in: fetch the addend first so its latency overlaps the TMEM drain
        uint4 addv[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
        if (MODE == DGRAD && a.accumulate) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int col = n0 + cb + (((k * 32 + lane) & 1) * 8);
                if (rowp[k] >= 0 && col + 8 <= lim && (lim & 7) == 0)
                    addv[k] = *reinterpret_cast<const uint4*>(static_cast<const __half*>(a.addend) + rowp[k] + col);
            }
        }
        uint32_t v[16];
        tmem_ld16(tacc + (static_cast<uint32_t>(q * 32) << 16) + cb, v);
        if (cb + 16 >= BN) {
            // accumulator fully drained into registers: hand it back to the MMA
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_acc);
        }
        if (nk == 0) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0u;
        }
        // stage row `lane` (16 fp32 = 4 x 16 B slots, XOR-swizzled: conflict-free)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int slot = j ^ ((lane >> 1) & 3);
            *reinterpret_cast<float4*>(stg + lane * 16 + slot * 4) =
                make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                            __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        }
        __syncwarp();
        const int col0 = n0 + cb;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int idx = k * 32 + lane;
            const int r = idx >> 1, c8 = idx & 1;  // row, 8-column chunk
            const int j0 = 2 * c8, sw = (r >> 1) & 3;
            const float4 f0 = *reinterpret_cast<const float4*>(stg + r * 16 + ((j0 ^ sw) * 4));
            const float4 f1 = *reinterpret_cast<const float4*>(stg + r * 16 + (((j0 + 1) ^ sw) * 4));
            const int col = col0 + c8 * 8;
            if (rowp[k] < 0 || col >= lim) continue;
            float f[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
            if (MODE == WGRAD) {
                float* o = static_cast<float*>(a.out) + rowp[k] + col;
                if (col + 8 <= lim && (lim & 3) == 0) {
                    *reinterpret_cast<float4*>(o) = f0;
                    *reinterpret_cast<float4*>(o + 4) = f1;
                } else {
                    for (int e = 0; e < 8 && col + e < lim; ++e) o[e] = f[e];
                }
            } else {
                __half* o = static_cast<__half*>(a.out) + rowp[k] + col;
                if (col + 8 <= lim && (lim & 7) == 0) {
                    if (MODE == DGRAD && a.accumulate) {
                        const __half* oh = reinterpret_cast<const __half*>(&addv[k]);
#pragma unroll
                        for (int e = 0; e < 8; ++e) f[e] += __half2float(oh[e]);
                    }
                    uint4 pk;
                    __half2* p2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
                    for (int e = 0; e < 4; ++e) p2[e] = __floats2half2_rn(f[2 * e], f[2 * e + 1]);
                    *reinterpret_cast<uint4*>(o) = pk;
                } else {
                    for (int e = 0; e < 8 && col + e < lim; ++e) {
                        float x = f[e];
                        if (MODE == DGRAD && a.accumulate)
                            x += __half2float(static_cast<const __half*>(a.addend)[rowp[k] + col + e]);
                        o[e] = __float2half_rn(x);
                    }
                }
            }
        }
        __syncwarp();
    }
}

// Persistent, warp-specialised tcgen05 implicit GEMM.
//   warps 0-3 : producers (implicit-im2col gathers with cp.async, 16 B chunks)
//   warp  4   : MMA issuer (one elected lane) + TMEM owner
//   warps 5-8 : epilogue (tcgen05.ld -> regs -> swizzled smem staging -> coalesced stores)
// Two TMEM accumulators (2 x BN columns): the epilogue of tile i drains one
// while the MMA of tile i+1 fills the other, so stores overlap the mainloop.
// Tiles are strided over a grid of (SMs x CTAs/SM), m fastest (CTAs resident
// together share the same filter tile in L2).
template <int MODE, int BN, int ST>
struct TcPCfg {
    static constexpr int kABytes = kBM * kBK * 2;
    static constexpr int kBBytes = BN * kBK * 2;
    static constexpr int kStage = kABytes + kBBytes;
    static constexpr int kStaging = 4 * 32 * 16 * 4;  // 4 epilogue warps x 32 rows x 16 fp32
    static constexpr int kSmem = ST * kStage + kStaging + 1024 + 512;
    static constexpr bool kAMN = MODE == WGRAD;
    static constexpr bool kBMN = MODE == DGRAD || MODE == WGRAD;
    static constexpr int kThreads = 288;
};

template <int MODE, int BN, int ST>
__global__ void __launch_bounds__(288, (BN <= 128) ? 2 : 1)
    conv_tc_kernel(ConvArgs a, int tiles_m, int tiles_n, int n_tiles, const __grid_constant__ TmaDesc tma) {
    using Cfg = TcPCfg<MODE, BN, ST>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* gbase = smem_raw + (base - raw);
    float* staging = reinterpret_cast<float*>(gbase + ST * Cfg::kStage);
    uint64_t* full = reinterpret_cast<uint64_t*>(gbase + ST * Cfg::kStage + Cfg::kStaging);
    uint64_t* empty = full + ST;
    uint64_t* tfull = empty + ST;   // [2]
    uint64_t* tempty = tfull + 2;   // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nkb_total = (a.KG + kBK - 1) / kBK;

    // the dense operand arrives by TMA (fprop B, wgrad A, dgrad B when K % 64 == 0):
    // one extra arrive.expect_tx per stage on top of the 128 cp.async arrivals
    const bool use_tma = MODE == FPROP || MODE == WGRAD || (MODE == DGRAD && a.tma_b);
    if (tid == 0) {
        prefetch_tmap(&tma.m);
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], use_tma ? 129 : 128);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_fence_init();
    }
    if (warp == 4) tmem_alloc(tmem_slot, 2 * BN);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto tile_coords = [&](int t, int& m0, int& n0, int& kb0, int& nk) {
        const int tm = t % tiles_m;
        const int rest = t / tiles_m;
        const int tn = rest % tiles_n;
        const int split = rest / tiles_n;
        m0 = tm * kBM;
        n0 = tn * BN;
        kb0 = MODE == WGRAD ? split * a.kb_per_split : 0;
        nk = MODE == WGRAD ? max(0, min(a.kb_per_split, nkb_total - kb0)) : nkb_total;
    };

    if (warp < 4) {
        int it = 0;  // global k-block counter (stage/phase continue across tiles)
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
            int m0, n0, kb0, nk;
            tile_coords(t, m0, n0, kb0, nk);
// ------------------------------------------------ producers
            // All per-row / per-column address arithmetic is hoisted out of the
            // k loop: per k-block each thread does at most one tap decomposition,
            // and every chunk is a pointer add + bounds test (the instruction
            // budget per k-block must stay below the MMA time of the k-block).
            const __half* X = static_cast<const __half*>(a.x);
            const __half* Wt = static_cast<const __half*>(a.w);
            const int HoWo = a.Ho * a.Wo;
            constexpr int kBChunksPerRow = BN / 8;           // MN-major B: chunks per k row
            constexpr int kBRowStep = 128 / kBChunksPerRow;  // k rows advanced per i
            // A rows (fprop/dgrad): per-row image/base coordinates
            int rowN[8], rowY[8], rowX[8];
            if (MODE == FPROP || MODE == DGRAD) {
    #pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int m = m0 + (tid >> 3) + 16 * i;
                    if (m < a.M) {
                        if (MODE == FPROP) {
                            const int n = m / HoWo, rem = m - n * HoWo, oh = rem / a.Wo, ow = rem - oh * a.Wo;
                            rowN[i] = n;
                            rowY[i] = oh * a.stride - a.pad;
                            rowX[i] = ow * a.stride - a.pad;
                        } else {
                            const int HpWp = a.Hp * a.Wp;
                            const int n = m / HpWp, rem = m - n * HpWp, i2 = rem / a.Wp, j2 = rem - i2 * a.Wp;
                            rowN[i] = n;
                            // (h + p - r0) / st is exact: h = ph + st*i2 and r0 = (ph + p) mod st
                            rowY[i] = (a.ph + a.stride * i2 + a.pad - a.r0) / a.stride;
                            rowX[i] = (a.pw + a.stride * j2 + a.pad - a.q0) / a.stride;
                        }
                    } else {
                        rowN[i] = -1;
                        rowY[i] = rowX[i] = -(1 << 28);
                    }
                }
            }
            // fprop B: filter row offsets
            int64_t brow[BN / 16];
            if (MODE == FPROP) {
    #pragma unroll
                for (int i = 0; i < BN / 16; ++i) {
                    const int j = n0 + (tid >> 3) + 16 * i;
                    brow[i] = j < a.NG ? static_cast<int64_t>(j) * a.KG : -1;
                }
            }
            // dgrad B (MN-major filter [c][(tap,kout)]) and wgrad A/B: fixed column chunk
            const int mcB = tid % kBChunksPerRow;
            const int krowB = tid / kBChunksPerRow;
            const int64_t RSC = static_cast<int64_t>(a.R) * a.S * a.C;
            const bool dg_fast = (a.K % kBK) == 0;
            int wg_r = 0, wg_s = 0, wg_c = 0;
            bool wg_ok = false;
            if (MODE == WGRAD) {
                const int col = n0 + mcB * 8;
                wg_ok = col < a.NG;
                const int tap = col / a.C;
                wg_c = col - tap * a.C;
                wg_r = tap / a.S;
                wg_s = tap - wg_r * a.S;
            }

            for (int k = 0; k < nk; ++k, ++it) {
                const int s = it % ST;
                if (it >= ST) mbar_wait(&empty[s], ((it / ST) - 1) & 1);
                const uint32_t sa = base + s * Cfg::kStage;
                const uint32_t sb = sa + Cfg::kABytes;
                const int kb = kb0 + k;
                if (MODE == FPROP) {
                    const int kg = kb * kBK + 8 * (tid & 7);
                    const bool kok = kg < a.KG;
                    const int tap = kg / a.C, c = kg - tap * a.C;
                    const int r = tap / a.S, q = tap - r * a.S;
    #pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int row = (tid >> 3) + 16 * i;
                        const int ih = rowY[i] + r, iw = rowX[i] + q;
                        const bool ok = kok && static_cast<unsigned>(ih) < static_cast<unsigned>(a.H) &&
                                        static_cast<unsigned>(iw) < static_cast<unsigned>(a.W);
                        const __half* src = ok ? X + ((static_cast<int64_t>(rowN[i]) * a.H + ih) * a.W + iw) * a.C + c : X;
                        cp_async16(sa + kmaj_off(row, tid & 7), src, ok ? 16u : 0u);
                    }
                    // B: the filter tile [BN rows][64 k] in one TMA box (zero-filled out of range)
                    if (tid == 0) {
                        mbar_arrive_expect_tx(&full[s], BN * kBK * 2);
                        tma_load_2d(sb, &tma.m, &full[s], kb * kBK, n0);
                    }
                } else if (MODE == DGRAD) {
                    // A: DY gather, k-major over kg = tap*K + kout
                    const int kg = kb * kBK + 8 * (tid & 7);
                    const bool kok = kg < a.KG;
                    const int t = kg / a.K, kout = kg - t * a.K;
                    const int ti = t / a.nq, tq = t - ti * a.nq;
    #pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int row = (tid >> 3) + 16 * i;
                        const int oh = rowY[i] - ti, ow = rowX[i] - tq;
                        const bool ok = kok && rowN[i] >= 0 && static_cast<unsigned>(oh) < static_cast<unsigned>(a.Ho) &&
                                        static_cast<unsigned>(ow) < static_cast<unsigned>(a.Wo);
                        const __half* src =
                            ok ? X + ((static_cast<int64_t>(rowN[i]) * a.Ho + oh) * a.Wo + ow) * a.K + kout : X;
                        cp_async16(sa + kmaj_off(row, tid & 7), src, ok ? 16u : 0u);
                    }
                    // B: filter as MN-major [c][kg]
                    const int c = n0 + mcB * 8;
                    const bool cok = c < a.NG;
                    if (a.tma_b) {
                        // one 3-D box [64 kout][1 tap][64 c] per 64-channel MN atom
                        if (tid == 0) {
                            const int kg0 = kb * kBK;
                            const int t2 = kg0 / a.K, kbk = kg0 - t2 * a.K;
                            const int r2 = a.r0 + a.stride * (t2 / a.nq), q2 = a.q0 + a.stride * (t2 % a.nq);
                            mbar_arrive_expect_tx(&full[s], BN * kBK * 2);
#pragma unroll
                            for (int g = 0; g < BN / 64; ++g)
                                tma_load_3d(sb + g * 8192, &tma.m, &full[s], n0 + 64 * g, r2 * a.S + q2, kbk);
                        }
                    } else if (dg_fast) {
                        // the whole k-block lies in one tap: kout = kbk + krow
                        const int kg0 = kb * kBK;
                        const int t2 = kg0 / a.K, kbk = kg0 - t2 * a.K;
                        const int r2 = a.r0 + a.stride * (t2 / a.nq), q2 = a.q0 + a.stride * (t2 % a.nq);
                        const bool tok = kg0 < a.KG && cok;
                        const __half* bsrc = Wt + static_cast<int64_t>(kbk + krowB) * RSC + (r2 * a.S + q2) * a.C + c;
    #pragma unroll
                        for (int i = 0; i < BN / 16; ++i) {
                            const int krow = krowB + kBRowStep * i;
                            cp_async16(sb + mnmaj_off(mcB, krow, BN), tok ? bsrc + kBRowStep * i * RSC : Wt, tok ? 16u : 0u);
                        }
                    } else {
    #pragma unroll
                        for (int i = 0; i < BN / 16; ++i) {
                            const int krow = krowB + kBRowStep * i;
                            const int kg2 = kb * kBK + krow;
                            const bool ok = kg2 < a.KG && cok;
                            const int t2 = kg2 / a.K, ko2 = kg2 - t2 * a.K;
                            const int r2 = a.r0 + a.stride * (t2 / a.nq), q2 = a.q0 + a.stride * (t2 % a.nq);
                            const __half* src = ok ? Wt + ((static_cast<int64_t>(ko2) * a.R + r2) * a.S + q2) * a.C + c : Wt;
                            cp_async16(sb + mnmaj_off(mcB, krow, BN), src, ok ? 16u : 0u);
                        }
                    }
                } else {
                    // WGRAD. A = DY^T as MN-major [kout][m]: two TMA boxes [64 pixels][64 kout]
                    if (tid == 0) {
                        mbar_arrive_expect_tx(&full[s], kBM * kBK * 2);
                        tma_load_2d(sa, &tma.m, &full[s], m0, kb * kBK);
                        tma_load_2d(sa + 8192, &tma.m, &full[s], m0 + 64, kb * kBK);
                    }
                    // B = im2col(X)^T as MN-major [(r,s,c)][m]; pixel walk is incremental
                    {
                        int m = kb * kBK + krowB;
                        int n = m / HoWo;
                        int rem = m - n * HoWo;
                        int oh = rem / a.Wo, ow = rem - oh * a.Wo;
    #pragma unroll
                        for (int i = 0; i < BN / 16; ++i) {
                            const int krow = krowB + kBRowStep * i;
                            const int ih = oh * a.stride - a.pad + wg_r, iw = ow * a.stride - a.pad + wg_s;
                            const bool ok = wg_ok && m < a.KG && static_cast<unsigned>(ih) < static_cast<unsigned>(a.H) &&
                                            static_cast<unsigned>(iw) < static_cast<unsigned>(a.W);
                            const __half* src = ok ? X + ((static_cast<int64_t>(n) * a.H + ih) * a.W + iw) * a.C + wg_c : X;
                            cp_async16(sb + mnmaj_off(mcB, krow, BN), src, ok ? 16u : 0u);
                            m += kBRowStep;
                            ow += kBRowStep;
                            while (ow >= a.Wo) {
                                ow -= a.Wo;
                                if (++oh == a.Ho) {
                                    oh = 0;
                                    ++n;
                                }
                            }
                        }
                    }
                }
                // the mbarrier arrival fires when THIS thread's copies of the stage
                // land; the producer never blocks on its own loads
                cp_async_mbar_arrive_noinc(&full[s]);
            }
        }
        cp_async_wait<0>();
    } else if (warp == 4) {
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_f16(kBM, BN, Cfg::kAMN ? 1 : 0, Cfg::kBMN ? 1 : 0);
            int it = 0, lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                int m0, n0, kb0, nk;
                tile_coords(t, m0, n0, kb0, nk);
                const int acc = lt & 1;
                mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t dcol = tmem + acc * BN;
                for (int k = 0; k < nk; ++k, ++it) {
                    const int s = it % ST;
                    mbar_wait(&full[s], (it / ST) & 1);
                    tc_fence_after();
                    const uint32_t sa = base + s * Cfg::kStage;
                    const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        // TMA-loaded MN-major operands: 8 KB per 64-element MN atom (LBO),
                        // 1 KB per 8 k-rows (SBO); cp.async MN-major B interleaves the atoms
                        const uint64_t ad = Cfg::kAMN ? umma_desc_sw128(sa + kk * 2048, 8192, 1024)
                                                      : umma_desc_sw128(sa + kk * 32, 16, 1024);
                        const uint64_t bd =
                            !Cfg::kBMN ? umma_desc_sw128(sb + kk * 32, 16, 1024)
                            : (MODE == DGRAD && a.tma_b)
                                ? umma_desc_sw128(sb + kk * 2048, 8192, 1024)
                                : umma_desc_sw128(sb + kk * 2 * (BN / 64) * 1024, 1024, (BN / 64) * 1024);
                        umma_f16(dcol, ad, bd, idesc, (k > 0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(&tfull[acc]);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ epilogue warps 5..8
        float* stg = staging + (warp - 5) * 32 * 16;
        int lt = 0;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
            int m0, n0, kb0, nk;
            tile_coords(t, m0, n0, kb0, nk);
            const int acc = lt & 1;
            mbar_wait(&tfull[acc], (lt >> 1) & 1);
            tc_fence_after();
            epilogue_tile<MODE, BN>(a, t / (tiles_m * tiles_n), m0, n0, nk, tmem + acc * BN, warp & 3, lane, stg,
                                    &tempty[acc]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc(tmem, 2 * BN);
    }
}

// Epilogue v2 (all-TMA kernel): warp w drains TMEM lane quadrant q = w & 3
// (tile rows 32q..32q+31) over columns [c_lo, c_lo + NCOL), SC columns per
// step: tcgen05.ld -> XOR-swizzled smem staging (row = lane, SC/4 slots of
// 16 B) -> coalesced 16-byte stores (SC/8 lanes per row).  The dgrad residual
// addend of step j+1 is loaded while step j is stored, so its global latency
// hides behind the TMEM drain instead of being exposed at every step.
template <int SC>
SDB_DEV void tmem_ld_cols(uint32_t taddr, uint32_t (&v)[SC]);
template <>
SDB_DEV void tmem_ld_cols<16>(uint32_t taddr, uint32_t (&v)[16]) { tmem_ld16(taddr, v); }
template <>
SDB_DEV void tmem_ld_cols<32>(uint32_t taddr, uint32_t (&v)[32]) { tmem_ld32(taddr, v); }

// f32 + f16 -> f32 with one rounding (sm_100 mixed-precision add)
SDB_DEV float fadd_f16(uint16_t h, float c) {
    float r;
    asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(r) : "h"(h), "f"(c));
    return r;
}
SDB_DEV uint32_t pack_half2(float lo, float hi) {
    const __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}
// backward of the leaky / ReLU that produced y, on a pair of rounded fp16
// gradients p: y > 0 ? p : rn16(f32(p) * neg)  (neg2 = neg in both halves of a
// f32x2), exactly the scalar float expression, in 5 instructions per pair
SDB_DEV uint32_t leaky_mask_half2(uint32_t p, uint32_t y, uint64_t neg2) {
    const __half2 ph = *reinterpret_cast<const __half2*>(&p);
    const float2 pf = __half22float2(ph);
    const uint64_t pf2 = static_cast<uint64_t>(__float_as_uint(pf.x)) |
                         (static_cast<uint64_t>(__float_as_uint(pf.y)) << 32);
    uint64_t q2;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(q2) : "l"(pf2), "l"(neg2));
    const uint32_t q = pack_half2(__uint_as_float(static_cast<uint32_t>(q2)), __uint_as_float(static_cast<uint32_t>(q2 >> 32)));
    const uint32_t m = __hgt2_mask(*reinterpret_cast<const __half2*>(&y), __float2half2_rn(0.f));
    return (p & m) | (q & ~m);
}

template <int MODE, int NCOL, int SC, bool ADD, bool MSK>
SDB_DEV void epilogue_tile_v2(const ConvArgs& a, int split, int m0, int n0, int nk, uint32_t tacc, int q, int lane,
                              int c_lo, float* stg, uint64_t* tfull_acc, uint32_t tfull_phase, uint64_t* tempty_acc) {
    constexpr int NSTEP = NCOL / SC;
    constexpr int LPR = SC / 8;        // lanes per row in the store phase
    constexpr int NK = LPR;            // store rows per lane = 32 / (32 / LPR)
    constexpr int SLOTS = SC / 4;      // 16-byte slots per staged row
    int64_t rowp[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        const int r = (k * 32 + lane) / LPR;
        const int grow = m0 + q * 32 + r;
        int64_t o = -1;
        if (grow < a.M) {
            if (MODE == FPROP) {
                o = static_cast<int64_t>(grow) * a.NG;
            } else if (MODE == DGRAD) {
                if (a.stride == 1) {
                    // one phase covering the whole input grid: GEMM row = input pixel
                    o = static_cast<int64_t>(grow) * a.C;
                } else {
                    const int HpWp = a.Hp * a.Wp;
                    const int n = grow / HpWp, rem = grow - n * HpWp, i2 = rem / a.Wp, j2 = rem - i2 * a.Wp;
                    o = ((static_cast<int64_t>(n) * a.H + a.ph + a.stride * i2) * a.W + a.pw + a.stride * j2) * a.C;
                }
            } else {
                o = (static_cast<int64_t>(split) * a.M + grow) * a.NG;
            }
        }
        rowp[k] = o;
    }
    const int lim = MODE == DGRAD ? a.C : a.NG;
    const bool vec = MODE == WGRAD ? (lim & 3) == 0 : (lim & 7) == 0;
    constexpr bool add = MODE == DGRAD && ADD;
    constexpr bool msk = MODE == DGRAD && MSK;
    const int c8 = lane % LPR;
    // dgrad residual addend / activation mask: a 3-deep register ring over the
    // (fully unrolled) column steps, two steps loaded ahead; the first two are
    // issued before the accumulator is even ready
    uint4 addb[3][NK], mskb[3][NK];
    auto load_vec = [&](const void* src, uint4 (&dst)[NK], int cb) {
        const int col = n0 + c_lo + cb + c8 * 8;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
            dst[k] = make_uint4(0, 0, 0, 0);
            if (rowp[k] >= 0 && col + 8 <= lim && vec)
                dst[k] = *reinterpret_cast<const uint4*>(static_cast<const __half*>(src) + rowp[k] + col);
        }
    };
    auto prefetch = [&](int js) {
        if (js >= NSTEP) return;
        if (add) load_vec(a.addend, addb[js % 3], js * SC);
        if (msk) load_vec(a.mask, mskb[js % 3], js * SC);
    };
    const uint64_t neg2 = static_cast<uint64_t>(__float_as_uint(a.mask_neg)) * 0x100000001ull;
    prefetch(0);
    prefetch(1);
    mbar_wait(tfull_acc, tfull_phase);
    tc_fence_after();
#pragma unroll
    for (int js = 0; js < NSTEP; ++js) {
        const int cb = js * SC;
        prefetch(js + 2);
        const uint4* addv = addb[js % 3];
        const uint4* mskv = mskb[js % 3];
        uint32_t v[SC];
        tmem_ld_cols<SC>(tacc + (static_cast<uint32_t>(q * 32) << 16) + c_lo + cb, v);
        if (cb + SC >= NCOL) {
            // this warp's part of the accumulator is in registers: release it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_acc);
        }
        if (nk == 0) {
#pragma unroll
            for (int j = 0; j < SC; ++j) v[j] = 0u;
        }
#pragma unroll
        for (int j = 0; j < SLOTS; ++j) {
            const int slot = j ^ (lane & (SLOTS - 1));
            *reinterpret_cast<float4*>(stg + lane * SC + slot * 4) =
                make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]), __uint_as_float(v[4 * j + 2]),
                            __uint_as_float(v[4 * j + 3]));
        }
        __syncwarp();
        const int col = n0 + c_lo + cb + c8 * 8;
        // all staged reads first (independent LDS in flight), then the stores
        float4 fa[NK], fb[NK];
#pragma unroll
        for (int k = 0; k < NK; ++k) {
            const int r = (k * 32 + lane) / LPR;
            const int sw = r & (SLOTS - 1);
            fa[k] = *reinterpret_cast<const float4*>(stg + r * SC + (((2 * c8) ^ sw) * 4));
            fb[k] = *reinterpret_cast<const float4*>(stg + r * SC + (((2 * c8 + 1) ^ sw) * 4));
        }
#pragma unroll
        for (int k = 0; k < NK; ++k) {
            const float4 f0 = fa[k], f1 = fb[k];
            if (rowp[k] < 0 || col >= lim) continue;
            float f[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
            if (MODE == WGRAD) {
                float* o = static_cast<float*>(a.out) + rowp[k] + col;
                if (col + 8 <= lim && vec) {
                    *reinterpret_cast<float4*>(o) = f0;
                    *reinterpret_cast<float4*>(o + 4) = f1;
                } else {
                    for (int e = 0; e < 8 && col + e < lim; ++e) o[e] = f[e];
                }
            } else {
                __half* o = static_cast<__half*>(a.out) + rowp[k] + col;
                if (col + 8 <= lim && vec) {
                    // per pair: s = acc + addend (mixed-precision add, one rounding),
                    // p = rn16(s); masked: out = y > 0 ? p : rn16(f32(p) * neg)
                    uint32_t pk[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float s0 = f[2 * e], s1 = f[2 * e + 1];
                        if (add) {
                            const uint32_t h2 = reinterpret_cast<const uint32_t*>(&addv[k])[e];
                            s0 = fadd_f16(static_cast<uint16_t>(h2 & 0xffffu), s0);
                            s1 = fadd_f16(static_cast<uint16_t>(h2 >> 16), s1);
                        }
                        pk[e] = pack_half2(s0, s1);
                        if (msk) pk[e] = leaky_mask_half2(pk[e], reinterpret_cast<const uint32_t*>(&mskv[k])[e], neg2);
                    }
                    *reinterpret_cast<uint4*>(o) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                } else {
                    for (int e = 0; e < 8 && col + e < lim; ++e) {
                        float x = f[e];
                        if (add) x += __half2float(static_cast<const __half*>(a.addend)[rowp[k] + col + e]);
                        if (msk) {
                            x = __half2float(__float2half_rn(x));
                            if (!(__half2float(static_cast<const __half*>(a.mask)[rowp[k] + col + e]) > 0.f))
                                x = __fmul_rn(a.mask_neg, x);
                        }
                        o[e] = __float2half_rn(x);
                    }
                }
            }
        }
        __syncwarp();
    }
}

// Epilogue v3 (fp16 output through TMA stores): the warp's TMEM lane quadrant
// is read with tcgen05.ld (lane = tile row, SC consecutive columns), packed to
// fp16 in registers and written row-per-lane into a swizzled staging box
// (SWIZZLE_64B for 64-byte rows, SWIZZLE_32B for 32-byte rows: conflict-free),
// which one lane hands to the TMA engine (cp.async.bulk.tensor store).  Two
// staging boxes per warp alternate, so the store of step j overlaps step j+1;
// partial tiles are clipped by the tensor map bounds.
// Column statistics of a staged fp16 box (rows = lanes of the quadrant): lane
// L sums column L (SC = 32) or half a column (SC = 16: lanes 16-31 take rows
// 16-31, folded in by one shuffle) -- every value widened to FP64 and its
// square formed exactly, like the statistics kernel (src/syncbn.cpp:29-39).
template <int SC>
SDB_DEV void box_column_stats(const uint8_t* buf, int lane, double& S, double& Q) {
    constexpr int ROWB = SC * 2;
    const int col = SC == 32 ? lane : (lane & 15);
    const int r0 = SC == 32 ? 0 : (lane >> 4) * 16;
    constexpr int NR = SC == 32 ? 32 : 16;
    double s = 0.0, qq = 0.0;
#pragma unroll 8
    for (int rr = 0; rr < NR; ++rr) {
        const int r = r0 + rr;
        const int j = col >> 3;
        const int pj = SC == 32 ? (j ^ ((r >> 1) & 3)) : (j ^ ((r >> 2) & 1));
        const __half h = *reinterpret_cast<const __half*>(buf + r * ROWB + pj * 16 + (col & 7) * 2);
        const double x = static_cast<double>(__half2float(h));
        s = __dadd_rn(s, x);
        qq = __fma_rn(x, x, qq);
    }
    if (SC == 16) {
        const double so = __shfl_down_sync(0xffffffffu, s, 16), qo = __shfl_down_sync(0xffffffffu, qq, 16);
        s = __dadd_rn(s, so);
        qq = __dadd_rn(qq, qo);
    }
    S = __dadd_rn(S, s);
    Q = __dadd_rn(Q, qq);
}

template <int NCOL, int SC>
SDB_DEV void epilogue_tile_tmastore(const CUtensorMap* omap, int m0, int n0, int nk, uint32_t tacc, int q, int lane,
                                    int c_lo, uint8_t* stg, uint64_t* tfull_acc, uint32_t tfull_phase,
                                    uint64_t* tempty_acc, int& sb, double* cs = nullptr) {
    constexpr int NSTEP = NCOL / SC;
    constexpr int ROWB = SC * 2;
    constexpr int BUFB = 32 * ROWB;
    mbar_wait(tfull_acc, tfull_phase);
    tc_fence_after();
#pragma unroll
    for (int js = 0; js < NSTEP; ++js) {
        uint32_t v[SC];
        tmem_ld_cols<SC>(tacc + (static_cast<uint32_t>(q * 32) << 16) + c_lo + js * SC, v);
        if (js == NSTEP - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_acc);
        }
        if (nk == 0) {
#pragma unroll
            for (int j = 0; j < SC; ++j) v[j] = 0u;
        }
        // the box about to be overwritten was handed to the TMA two steps ago
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        uint8_t* buf = stg + sb * BUFB;
#pragma unroll
        for (int j = 0; j < SC / 8; ++j) {
            const uint4 pk = make_uint4(pack_half2(__uint_as_float(v[8 * j]), __uint_as_float(v[8 * j + 1])),
                                        pack_half2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                                        pack_half2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                                        pack_half2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
            const int pj = SC == 32 ? (j ^ ((lane >> 1) & 3)) : (j ^ ((lane >> 2) & 1));
            *reinterpret_cast<uint4*>(buf + lane * ROWB + pj * 16) = pk;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            tma_store_2d(omap, smem_u32(buf), n0 + c_lo + js * SC, m0 + q * 32);
            bulk_commit();
        }
        // rows beyond M hold zeros (TMA zero-fills the A operand), adding +0.0
        if (cs) box_column_stats<SC>(buf, lane, cs[2 * js], cs[2 * js + 1]);
        sb ^= 1;
    }
}

// Epilogue v4 (stride-1 dgrad with the residual addend and a sign-bitmap
// mask, BN = 256): lane = tile row as in v3.  The addend box of each column
// step arrives by TMA into a two-slot ring (issued two steps ahead, the first
// two before the accumulator is ready), the 32 mask bits of the row are one
// 4-byte load, and the result leaves by TMA store:
//   out = m ? p : rn16(f32(p) * neg),  p = rn16(acc + addend)
template <int NCOL, int SC>
SDB_DEV void epilogue_tile_resid(const ConvArgs& a, const CUtensorMap* omap, const CUtensorMap* rmap, int m0, int n0,
                                 int nk, uint32_t tacc, int q, int lane, int c_lo, uint8_t* ostg, uint8_t* rstg,
                                 uint64_t* rbar, uint64_t* tfull_acc, uint32_t tfull_phase, uint64_t* tempty_acc,
                                 int& sb) {
    static_assert(SC == 32, "residual epilogue: 64-byte rows");
    constexpr int NSTEP = NCOL / SC;
    constexpr int ROWB = SC * 2;
    constexpr int BUFB = 32 * ROWB;
    static_assert(NSTEP % 2 == 0, "two-slot ring: slot = step & 1");
    const int row = m0 + q * 32 + lane;
    const int cbase = n0 + c_lo;
    auto issue = [&](int js) {
        if (lane == 0 && js < NSTEP) {
            uint64_t* bar = &rbar[js & 1];
            mbar_arrive_expect_tx(bar, BUFB);
            tma_load_2d(smem_u32(rstg + (js & 1) * BUFB), rmap, bar, cbase + js * SC, m0 + q * 32);
        }
    };
    issue(0);
    issue(1);
    // the row's mask bits for the whole tile (NCOL / 8 bytes)
    uint32_t mb[NSTEP];
    const int cb8 = a.C / 8;
#pragma unroll
    for (int js = 0; js < NSTEP; ++js)
        mb[js] = (row < a.M && cbase + js * SC < a.C)
                     ? *reinterpret_cast<const uint32_t*>(a.mbits + static_cast<int64_t>(row) * cb8 + (cbase + js * SC) / 8)
                     : 0u;
    const uint64_t neg2 = static_cast<uint64_t>(__float_as_uint(a.mask_neg)) * 0x100000001ull;
    mbar_wait(tfull_acc, tfull_phase);
    tc_fence_after();
#pragma unroll
    for (int js = 0; js < NSTEP; ++js) {
        uint32_t v[SC];
        tmem_ld_cols<SC>(tacc + (static_cast<uint32_t>(q * 32) << 16) + c_lo + js * SC, v);
        if (js == NSTEP - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_acc);
        }
        if (nk == 0) {
#pragma unroll
            for (int j = 0; j < SC; ++j) v[j] = 0u;
        }
        mbar_wait(&rbar[js & 1], (js >> 1) & 1);
        const uint8_t* rb = rstg + (js & 1) * BUFB + lane * ROWB;
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        uint8_t* buf = ostg + sb * BUFB;
#pragma unroll
        for (int j = 0; j < SC / 8; ++j) {
            const int pj = j ^ ((lane >> 1) & 3);
            const uint4 r4 = *reinterpret_cast<const uint4*>(rb + pj * 16);
            const uint32_t rw[4] = {r4.x, r4.y, r4.z, r4.w};
            uint32_t pk[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float s0 = fadd_f16(static_cast<uint16_t>(rw[e] & 0xffffu), __uint_as_float(v[8 * j + 2 * e]));
                const float s1 = fadd_f16(static_cast<uint16_t>(rw[e] >> 16), __uint_as_float(v[8 * j + 2 * e + 1]));
                const uint32_t p = pack_half2(s0, s1);
                const uint32_t b2 = mb[js] >> (8 * j + 2 * e);
                const uint32_t m = ((0u - (b2 & 1u)) & 0xffffu) | ((0u - ((b2 >> 1) & 1u)) & 0xffff0000u);
                const __half2 ph = *reinterpret_cast<const __half2*>(&p);
                const float2 pf = __half22float2(ph);
                const uint64_t pf2 = static_cast<uint64_t>(__float_as_uint(pf.x)) |
                                     (static_cast<uint64_t>(__float_as_uint(pf.y)) << 32);
                uint64_t q2;
                asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(q2) : "l"(pf2), "l"(neg2));
                const uint32_t qn = pack_half2(__uint_as_float(static_cast<uint32_t>(q2)),
                                               __uint_as_float(static_cast<uint32_t>(q2 >> 32)));
                pk[e] = (p & m) | (qn & ~m);
            }
            *reinterpret_cast<uint4*>(buf + lane * ROWB + pj * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
        // the addend slot is free again (all lanes read it): reload it two steps ahead
        fence_proxy_async();
        __syncwarp();
        issue(js + 2);
        if (lane == 0) {
            tma_store_2d(omap, smem_u32(buf), cbase + js * SC, m0 + q * 32);
            bulk_commit();
        }
        sb ^= 1;
    }
}

// Epilogue EPI 2 (stride-1 dgrad whose output feeds an InPlace-ABN backward):
// the plain TMA-store epilogue plus the layer's backward statistics.  The
// stored y box of each column step arrives by TMA into a two-slot ring (as
// the residual epilogue's addend); after the rounded fp16 dy box is staged,
// lane = column (SC = 32) or half a column (SC = 16) walks the 32 rows of both
// boxes and accumulates, in fp64 exactly like the statistics kernel,
//   S += dz,  Q += dz * xhat   (dz, xhat in float: stats_kernel KIND 2)
template <int NCOL, int SC>
SDB_DEV void epilogue_tile_bstats(const ConvArgs& a, const CUtensorMap* omap, const CUtensorMap* ymap, int m0, int n0,
                                  int nk, uint32_t tacc, int q, int lane, int c_lo, uint8_t* ostg, uint8_t* ystg,
                                  uint64_t* ybar, uint64_t* tfull_acc, uint32_t tfull_phase, uint64_t* tempty_acc,
                                  int& sb, double* cs) {
    constexpr int NSTEP = NCOL / SC;
    constexpr int ROWB = SC * 2;
    constexpr int BUFB = 32 * ROWB;
    // each ring slot is used NSTEP / 2 times per tile: an even count keeps the
    // barrier parity aligned with js at the start of every tile
    static_assert((NSTEP / 2) % 2 == 0, "two-slot ring parity");
    const int cbase = n0 + c_lo;
    auto issue = [&](int js) {
        if (lane == 0 && js < NSTEP) {
            uint64_t* bar = &ybar[js & 1];
            mbar_arrive_expect_tx(bar, BUFB);
            tma_load_2d(smem_u32(ystg + (js & 1) * BUFB), ymap, bar, cbase + js * SC, m0 + q * 32);
        }
    };
    issue(0);
    issue(1);
    const float slope = a.bs_slope, inv_slope = 1.0f / a.bs_slope;
    mbar_wait(tfull_acc, tfull_phase);
    tc_fence_after();
#pragma unroll
    for (int js = 0; js < NSTEP; ++js) {
        uint32_t v[SC];
        tmem_ld_cols<SC>(tacc + (static_cast<uint32_t>(q * 32) << 16) + c_lo + js * SC, v);
        if (js == NSTEP - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_acc);
        }
        if (nk == 0) {
#pragma unroll
            for (int j = 0; j < SC; ++j) v[j] = 0u;
        }
        // one output box (the smem budget keeps the mainloop's stages): the
        // previous step's store has had the statistics pass to drain it
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
        uint8_t* buf = ostg;
#pragma unroll
        for (int j = 0; j < SC / 8; ++j) {
            const uint4 pk = make_uint4(pack_half2(__uint_as_float(v[8 * j]), __uint_as_float(v[8 * j + 1])),
                                        pack_half2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                                        pack_half2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                                        pack_half2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
            const int pj = SC == 32 ? (j ^ ((lane >> 1) & 3)) : (j ^ ((lane >> 2) & 1));
            *reinterpret_cast<uint4*>(buf + lane * ROWB + pj * 16) = pk;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            tma_store_2d(omap, smem_u32(buf), cbase + js * SC, m0 + q * 32);
            bulk_commit();
        }
        // statistics over the staged dy box and the y box of the same rows
        mbar_wait(&ybar[js & 1], (js >> 1) & 1);
        const uint8_t* yb = ystg + (js & 1) * BUFB;
        {
            const int col = SC == 32 ? lane : (lane & 15);
            const int r0 = SC == 32 ? 0 : (lane >> 4) * 16;
            constexpr int NR = SC == 32 ? 32 : 16;
            const int gcol = cbase + js * SC + col;
            const bool ok = gcol < a.C;
            const float ig = ok ? 1.0f / a.bs_gamma[gcol] : 0.f;
            const float bt = ok ? a.bs_beta[gcol] : 0.f;
            double s = 0.0, qq = 0.0;
#pragma unroll 8
            for (int rr = 0; rr < NR; ++rr) {
                const int r = r0 + rr;
                const int j = col >> 3;
                const int pj = SC == 32 ? (j ^ ((r >> 1) & 3)) : (j ^ ((r >> 2) & 1));
                const int off = r * ROWB + pj * 16 + (col & 7) * 2;
                const float dyv = __half2float(*reinterpret_cast<const __half*>(buf + off));
                const float yv = __half2float(*reinterpret_cast<const __half*>(yb + off));
                const float z = yv >= 0.f ? yv : __fmul_rn(yv, inv_slope);
                const float dz = __fmul_rn(dyv, yv > 0.f ? 1.f : slope);
                const float xh = __fmul_rn(__fsub_rn(z, bt), ig);
                s = __dadd_rn(s, static_cast<double>(dz));
                qq = __fma_rn(static_cast<double>(dz), static_cast<double>(xh), qq);
            }
            if (SC == 16) {
                const double so = __shfl_down_sync(0xffffffffu, s, 16), qo = __shfl_down_sync(0xffffffffu, qq, 16);
                s = __dadd_rn(s, so);
                qq = __dadd_rn(qq, qo);
            }
            if (ok) {
                cs[2 * js] = __dadd_rn(cs[2 * js], s);
                cs[2 * js + 1] = __dadd_rn(cs[2 * js + 1], qq);
            }
        }
        // the y slot is free again (all lanes read it): reload it two steps ahead
        fence_proxy_async();
        __syncwarp();
        issue(js + 2);
    }
    (void)sb;
}

// ============================================================ all-TMA tcgen05 kernel
// Both operands arrive by TMA, the activation side through the im2col mode of
// cp.async.bulk.tensor (the hardware walks the output-pixel traversal of the
// convolution, applies the filter-tap offset and zero-fills the padding), so
// the whole mainloop of a stage is 1-6 TMA instructions from one thread:
//   fprop  A = im2col(X)        [128 pixels][64 c]   K-major   (needs C % 64 == 0)
//          B = W               [BN k][64 (r,s,c)]   K-major   2-D tile
//   dgrad  A = im2col(DY) over the sub-pixel phase grid, taps as non-negative
//              offsets from a shifted base          K-major   (needs K % 64 == 0)
//          B = W as [c][(tap,k)]                    MN-major  3-D tile
//   wgrad  computed transposed, DW^T[(r,s,c)][k] = sum_px im2col(X)[px][(r,s,c)] DY[px][k]:
//          A = im2col(X)^T      [64 px][128 (r,s,c)] MN-major  (needs C % 64 == 0)
//          B = DY^T             [64 px][BN k]        MN-major  2-D tile
//          so only 16 KB of each stage goes through the (slower) im2col path;
//          the fp32 split-K partials are [split][(r,s,c)][k] and the reduce
//          transposes them into the KRSC gradient.
// warp 0: TMA producer (one lane), warp 1: MMA issuer + TMEM owner,
// warps 2-5: epilogue (TMEM lane quadrant = warp & 3).
struct alignas(64) TmaPair {
    CUtensorMap a, b;
    CUtensorMap o;  // output [rows][cols] fp16, box {SC cols, 32 rows} (when ConvArgs::tma_out)
    CUtensorMap r;  // dgrad residual addend, same box (EPI 1)
};

SDB_DEV void tma_im2col_4d(uint32_t dst, const void* map, uint64_t* bar, int c, int w, int h, int n, int off_w,
                           int off_h) {
    const uint16_t ow = static_cast<uint16_t>(off_w), oh = static_cast<uint16_t>(off_h);
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
        "%6}], [%2], {%7, %8};" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
        : "memory");
}

// BN = 256: 8 epilogue warps (two per TMEM lane quadrant, 128 columns each,
// 32-column steps) -- or EW = 16 (four per quadrant, 64 columns each) for the
// fprops whose epilogue also reduces the norm statistics, which is then the
// longer half of the tile pipeline; BN <= 128: 4 warps, 16-column steps (two
// CTAs per SM).  EPI 1 (dgrad residual + bitmask epilogue, BN = 256): per
// epilogue warp two output staging boxes and a two-slot addend ring (4 x 2 KB)
template <int MODE, int BN, int ST, int EPI = 0, int EW = (BN == 256 ? 8 : 4)>
struct TmaCfg {
    static constexpr int kABytes = kBM * kBK * 2;
    static constexpr int kBBytes = BN * kBK * 2;
    static constexpr int kStage = kABytes + kBBytes;
    static constexpr int kEpiWarps = EW;
    static constexpr int kSC = BN == 256 ? 32 : 16;
    // EPI 1: 2 output boxes + 2 addend slots per warp; EPI 2: 1 output box + 2 y slots
    static constexpr int kStaging = EPI == 1 ? kEpiWarps * 4 * 32 * kSC * 2
                                  : EPI == 2 ? kEpiWarps * 3 * 32 * kSC * 2 : kEpiWarps * 32 * kSC * 4;
    static constexpr int kSmem = ST * kStage + kStaging + 1024 + 256;
    static constexpr int kThreads = 64 + 32 * kEpiWarps;
    static constexpr int kPerSM = BN <= 128 ? 2 : 1;
};

template <int MODE, int BN, int ST, int EPI = 0, int EW = (BN == 256 ? 8 : 4)>
__global__ void __launch_bounds__(TmaCfg<MODE, BN, ST, EPI, EW>::kThreads, (BN <= 128) ? 2 : 1)
    conv_tma_kernel(ConvArgs a, int tiles_m, int tiles_n, int n_tiles, const __grid_constant__ TmaPair tm) {
    using Cfg = TmaCfg<MODE, BN, ST, EPI, EW>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* gbase = smem_raw + (base - raw);
    float* staging = reinterpret_cast<float*>(gbase + ST * Cfg::kStage);
    uint64_t* full = reinterpret_cast<uint64_t*>(gbase + ST * Cfg::kStage + Cfg::kStaging);
    uint64_t* empty = full + ST;
    uint64_t* tfull = empty + ST;   // [2]
    uint64_t* tempty = tfull + 2;   // [2]
    uint64_t* rbar = tempty + 2;    // [kEpiWarps][2] addend ring (EPI 1)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + (EPI ? 2 * Cfg::kEpiWarps : 0));

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nkb_total = (a.KG + kBK - 1) / kBK;
    if (tid == 0) {
        prefetch_tmap(&tm.a);
        prefetch_tmap(&tm.b);
        if (a.tma_out) prefetch_tmap(&tm.o);
        if (EPI) prefetch_tmap(&tm.r);
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < (EPI ? 2 * Cfg::kEpiWarps : 0); ++i) mbar_init(&rbar[i], 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], Cfg::kEpiWarps);
        }
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 2 * BN);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // everything above overlapped the previous kernel's tail (PDL)
    pdl_wait();
    pdl_trigger();

    // Rasterisation: fprop/dgrad stream a large activation operand against a
    // small filter, so the N tiles of one M tile run on neighbouring CTAs at
    // the same time (each activation block is read from HBM once, the filter
    // stays in L2); m-fastest order re-read the activation tiles_n times
    // (727 MB of DRAM reads for a 103 MB input, res5 shortcut).  wgrad streams
    // both operands along K and keeps m-fastest order within a split.
    auto tile_coords = [&](int t, int& m0, int& n0, int& kb0, int& nk) {
        int tm_, tn, split;
        if (MODE == WGRAD) {
            tm_ = t % tiles_m;
            const int rest = t / tiles_m;
            tn = rest % tiles_n;
            split = rest / tiles_n;
        } else {
            tn = t % tiles_n;
            tm_ = t / tiles_n;
            split = 0;
        }
        m0 = tm_ * kBM;
        n0 = tn * BN;
        kb0 = MODE == WGRAD ? split * a.kb_per_split : 0;
        nk = MODE == WGRAD ? max(0, min(a.kb_per_split, nkb_total - kb0)) : nkb_total;
    };

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer
            // A single thread issues every TMA of the CTA, so its per-k-block
            // instruction latency must stay well below the MMA time of a
            // k-block (~512 cycles at BN = 256): all divisions are hoisted to
            // the tile and the k-block coordinates advance by carries.
            const int HoWo = a.Ho * a.Wo;
            // wgrad: a k-block is 64 consecutive output pixels; 64 = dn*HoWo + doh*Wo + dow
            const int dn = kBK / HoWo, drem = kBK - dn * HoWo, doh = drem / a.Wo, dow = drem - doh * a.Wo;
            int it = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                int m0, n0, kb0, nk;
                tile_coords(t, m0, n0, kb0, nk);
                // im2col base of the tile's first output pixel (fprop / dgrad)
                int bw = 0, bh = 0, bn = 0;
                if (MODE == FPROP) {
                    const int n = m0 / HoWo, rem = m0 - n * HoWo, oh = rem / a.Wo, ow = rem - oh * a.Wo;
                    bn = n;
                    bh = oh * a.stride - a.pad;
                    bw = ow * a.stride - a.pad;
                } else if (MODE == DGRAD) {
                    const int HpWp = a.Hp * a.Wp;
                    const int n = m0 / HpWp, rem = m0 - n * HpWp, i2 = rem / a.Wp, j2 = rem - i2 * a.Wp;
                    bn = n;
                    // DY row of phase pixel i2 for tap ti: i2 + cy - ti; base shifted by (nr-1) so the
                    // per-tap offset (nr-1-ti) is non-negative
                    bh = i2 + (a.ph + a.pad - a.r0) / a.stride - (a.nr - 1);
                    bw = j2 + (a.pw + a.pad - a.q0) / a.stride - (a.nq - 1);
                }
                // k-block coordinates at k = 0, advanced by carries below
                //   fprop: (r, q, c) of kg0 = kb*64          dgrad: (ti, tq, kout)
                //   wgrad: output pixel (n, oh, ow) of kb*64
                int c0 = 0, t0 = 0, t1 = 0;  // channel, tap row, tap col   (fprop / dgrad)
                int pn = 0, poh = 0, pow_ = 0;  // wgrad pixel
                int ar[2] = {0, 0}, aq[2] = {0, 0}, ac[2] = {0, 0};  // wgrad A chunks (tap row/col, channel)
                if (MODE == WGRAD) {
                    const int p0 = kb0 * kBK;
                    pn = p0 / HoWo;
                    const int rem = p0 - pn * HoWo;
                    poh = rem / a.Wo;
                    pow_ = rem - poh * a.Wo;
#pragma unroll
                    for (int g = 0; g < 2; ++g) {
                        int col = m0 + 64 * g;
                        if (col >= a.M) col = 0;  // beyond the filter: any valid box (rows discarded)
                        const int tap = col / a.C;
                        ac[g] = col - tap * a.C;
                        ar[g] = tap / a.S;
                        aq[g] = tap - ar[g] * a.S;
                    }
                }
                for (int k = 0; k < nk; ++k, ++it) {
                    const int s = it % ST;
                    if (it >= ST) mbar_wait(&empty[s], ((it / ST) - 1) & 1);
                    const uint32_t sa = base + s * Cfg::kStage;
                    const uint32_t sb = sa + Cfg::kABytes;
                    const int kg0 = (kb0 + k) * kBK;
                    mbar_arrive_expect_tx(&full[s], Cfg::kStage);
                    if (MODE == FPROP) {
                        if (a.plain) tma_load_2d(sa, &tm.a, &full[s], kg0, m0);
                        else tma_im2col_4d(sa, &tm.a, &full[s], c0, bw, bh, bn, t1, t0);
                        tma_load_2d(sb, &tm.b, &full[s], kg0, n0);
                        // next (r, q, c): c += 64 with carries into q then r
                        c0 += kBK;
                        if (c0 >= a.C) {
                            c0 = 0;
                            if (++t1 == a.S) {
                                t1 = 0;
                                ++t0;
                            }
                        }
                    } else if (MODE == DGRAD) {
                        // (t0, t1) = (ti, tq), c0 = kout
                        if (a.plain) tma_load_2d(sa, &tm.a, &full[s], c0, m0);
                        else tma_im2col_4d(sa, &tm.a, &full[s], c0, bw, bh, bn, a.nq - 1 - t1, a.nr - 1 - t0);
                        const int r2 = a.r0 + a.stride * t0, q2 = a.q0 + a.stride * t1;
#pragma unroll
                        for (int g = 0; g < BN / 64; ++g)
                            tma_load_3d(sb + g * 8192, &tm.b, &full[s], n0 + 64 * g, r2 * a.S + q2, c0);
                        c0 += kBK;
                        if (c0 >= a.K) {
                            c0 = 0;
                            if (++t1 == a.nq) {
                                t1 = 0;
                                ++t0;
                            }
                        }
                    } else {
                        const int h = poh * a.stride - a.pad, w = pow_ * a.stride - a.pad;
#pragma unroll
                        for (int g = 0; g < 2; ++g) {
                            if (a.plain) tma_load_2d(sa + g * 8192, &tm.a, &full[s], ac[g], kg0);
                            else tma_im2col_4d(sa + g * 8192, &tm.a, &full[s], ac[g], w, h, pn, aq[g], ar[g]);
                        }
#pragma unroll
                        for (int g = 0; g < BN / 64; ++g) tma_load_2d(sb + g * 8192, &tm.b, &full[s], n0 + 64 * g, kg0);
                        // next pixel block: + (dn, doh, dow) in mixed radix (N, Ho, Wo)
                        pow_ += dow;
                        poh += doh;
                        pn += dn;
                        if (pow_ >= a.Wo) {
                            pow_ -= a.Wo;
                            ++poh;
                        }
                        if (poh >= a.Ho) {
                            poh -= a.Ho;
                            ++pn;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------ MMA issuer
            constexpr bool kAMN = MODE == WGRAD;
            constexpr bool kBMN = MODE != FPROP;
            constexpr uint32_t idesc = umma_idesc_f16(kBM, BN, kAMN ? 1 : 0, kBMN ? 1 : 0);
            int it = 0, lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                int m0, n0, kb0, nk;
                tile_coords(t, m0, n0, kb0, nk);
                const int acc = lt & 1;
                mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t dcol = tmem + acc * BN;
                for (int k = 0; k < nk; ++k, ++it) {
                    const int s = it % ST;
                    mbar_wait(&full[s], (it / ST) & 1);
                    tc_fence_after();
                    const uint32_t sa = base + s * Cfg::kStage;
                    const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        // TMA MN-major operands: 8 KB per 64-element MN atom (LBO), 1 KB per 8 k rows (SBO)
                        const uint64_t ad = kAMN ? umma_desc_sw128(sa + kk * 2048, 8192, 1024)
                                                 : umma_desc_sw128(sa + kk * 32, 16, 1024);
                        const uint64_t bd = kBMN ? umma_desc_sw128(sb + kk * 2048, 8192, 1024)
                                                 : umma_desc_sw128(sb + kk * 32, 16, 1024);
                        umma_f16(dcol, ad, bd, idesc, (k > 0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(&tfull[acc]);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ epilogue warps 2..
        constexpr int kNCol = BN * 4 / Cfg::kEpiWarps;  // columns per warp
        const int ew = warp - 2;
        float* stg = staging + ew * 32 * Cfg::kSC;
        const int c_lo = (ew / 4) * kNCol;
        // the dgrad residual addend / activation mask are compile-time variants
        // (a lean epilogue is what keeps these warps ahead of the stores)
        auto run = [&](auto add_c, auto msk_c) {
            int lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                int m0, n0, kb0, nk;
                tile_coords(t, m0, n0, kb0, nk);
                const int acc = lt & 1;
                epilogue_tile_v2<MODE, kNCol, Cfg::kSC, decltype(add_c)::value, decltype(msk_c)::value>(
                    a, t / (tiles_m * tiles_n), m0, n0, nk, tmem + acc * BN, warp & 3, lane, c_lo, stg, &tfull[acc],
                    (lt >> 1) & 1, &tempty[acc]);
            }
        };
        using T_ = std::true_type;
        using F_ = std::false_type;
        if constexpr (EPI == 1) {
            int lt = 0, sb = 0;
            uint8_t* ostg = reinterpret_cast<uint8_t*>(staging) + ew * 4 * (32 * Cfg::kSC * 2);
            uint8_t* rstg = ostg + 2 * (32 * Cfg::kSC * 2);
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                int m0, n0, kb0, nk;
                tile_coords(t, m0, n0, kb0, nk);
                const int acc = lt & 1;
                epilogue_tile_resid<kNCol, Cfg::kSC>(a, &tm.o, &tm.r, m0, n0, nk, tmem + acc * BN, warp & 3, lane,
                                                     c_lo, ostg, rstg, rbar + 2 * ew, &tfull[acc], (lt >> 1) & 1,
                                                     &tempty[acc], sb);
            }
            if (lane == 0) bulk_wait_all();
            __syncwarp();
        } else if constexpr (EPI == 2) {
            int lt = 0, sb = 0;
            uint8_t* ostg = reinterpret_cast<uint8_t*>(staging) + ew * 3 * (32 * Cfg::kSC * 2);
            uint8_t* ystg = ostg + (32 * Cfg::kSC * 2);
            constexpr int kStep = kNCol / Cfg::kSC;
            double cs[2 * kStep];
#pragma unroll
            for (int j = 0; j < 2 * kStep; ++j) cs[j] = 0.0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                int m0, n0, kb0, nk;
                tile_coords(t, m0, n0, kb0, nk);
                const int acc = lt & 1;
                epilogue_tile_bstats<kNCol, Cfg::kSC>(a, &tm.o, &tm.r, m0, n0, nk, tmem + acc * BN, warp & 3, lane,
                                                      c_lo, ostg, ystg, rbar + 2 * ew, &tfull[acc], (lt >> 1) & 1,
                                                      &tempty[acc], sb, cs);
            }
            // stats[cta][quadrant][sum dz | sum dz*xhat][BN] (every tile of a CTA has the same n0)
            const int lanes = Cfg::kSC == 32 ? 32 : 16;
            if (lane < lanes) {
                double* o = a.stats + (static_cast<int64_t>(blockIdx.x) * 4 + (warp & 3)) * 2 * BN;
#pragma unroll
                for (int js = 0; js < kStep; ++js) {
                    o[c_lo + js * Cfg::kSC + lane] = cs[2 * js];
                    o[BN + c_lo + js * Cfg::kSC + lane] = cs[2 * js + 1];
                }
            }
            if (lane == 0) bulk_wait_all();
            __syncwarp();
        } else if (MODE != WGRAD && a.tma_out) {
            int lt = 0, sb = 0;
            uint8_t* stg8 = reinterpret_cast<uint8_t*>(stg);
            constexpr int kStep = kNCol / Cfg::kSC;
            double cs[2 * kStep];
#pragma unroll
            for (int j = 0; j < 2 * kStep; ++j) cs[j] = 0.0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                int m0, n0, kb0, nk;
                tile_coords(t, m0, n0, kb0, nk);
                const int acc = lt & 1;
                epilogue_tile_tmastore<kNCol, Cfg::kSC>(&tm.o, m0, n0, nk, tmem + acc * BN, warp & 3, lane, c_lo,
                                                        stg8, &tfull[acc], (lt >> 1) & 1, &tempty[acc], sb,
                                                        (MODE == FPROP && a.stats) ? cs : nullptr);
            }
            if (MODE == FPROP && a.stats) {
                // this CTA's column block: stats[cta][quadrant][sum | sumsq][BN] (the host
                // guarantees that every tile of a CTA has the same n0)
                const int lanes = Cfg::kSC == 32 ? 32 : 16;
                if (lane < lanes) {
                    double* o = a.stats + (static_cast<int64_t>(blockIdx.x) * 4 + (warp & 3)) * 2 * BN;
#pragma unroll
                    for (int js = 0; js < kStep; ++js) {
                        o[c_lo + js * Cfg::kSC + lane] = cs[2 * js];
                        o[BN + c_lo + js * Cfg::kSC + lane] = cs[2 * js + 1];
                    }
                }
            }
            if (lane == 0) bulk_wait_all();
            __syncwarp();
        } else if (MODE == DGRAD && a.accumulate && a.mask) run(T_{}, T_{});
        else if (MODE == DGRAD && a.accumulate) run(T_{}, F_{});
        else if (MODE == DGRAD && a.mask) run(F_{}, T_{});
        else run(F_{}, F_{});
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 2 * BN);
    }
}

// ============================================================ CUDA-core kernel
// Same GEMM views, scalar gathers, 64x64x16 tiles; fp32 or fp16 storage.
template <class T>
SDB_DEV float a_elem(const ConvArgs& a, int mode, int m, int kg) {
    const T* X = static_cast<const T*>(a.x);
    if (m >= a.M || kg >= a.KG) return 0.f;
    if (mode == FPROP) {
        const int HoWo = a.Ho * a.Wo;
        const int n = m / HoWo, rem = m - n * HoWo, oh = rem / a.Wo, ow = rem - oh * a.Wo;
        const int tap = kg / a.C, c = kg - tap * a.C, r = tap / a.S, q = tap - r * a.S;
        const int ih = oh * a.stride - a.pad + r, iw = ow * a.stride - a.pad + q;
        if (ih < 0 || ih >= a.H || iw < 0 || iw >= a.W) return 0.f;
        return to_f<T>(X[((static_cast<int64_t>(n) * a.H + ih) * a.W + iw) * a.C + c]);
    } else if (mode == DGRAD) {
        const int HpWp = a.Hp * a.Wp;
        const int n = m / HpWp, rem = m - n * HpWp, i2 = rem / a.Wp, j2 = rem - i2 * a.Wp;
        const int t = kg / a.K, kout = kg - t * a.K;
        const int r = a.r0 + a.stride * (t / a.nq), q = a.q0 + a.stride * (t % a.nq);
        const int yy = a.ph + a.stride * i2 + a.pad - r, xx = a.pw + a.stride * j2 + a.pad - q;
        if (yy < 0 || xx < 0) return 0.f;
        const int oh = yy / a.stride, ow = xx / a.stride;
        if (oh >= a.Ho || ow >= a.Wo) return 0.f;
        return to_f<T>(X[((static_cast<int64_t>(n) * a.Ho + oh) * a.Wo + ow) * a.K + kout]);
    } else {
        const T* DY = static_cast<const T*>(a.w);
        return to_f<T>(DY[static_cast<int64_t>(kg) * a.K + m]);  // A[kout][pixel]
    }
}

template <class T>
SDB_DEV float b_elem(const ConvArgs& a, int mode, int j, int kg) {
    if (j >= a.NG || kg >= a.KG) return 0.f;
    if (mode == FPROP) {
        return to_f<T>(static_cast<const T*>(a.w)[static_cast<int64_t>(j) * a.KG + kg]);
    } else if (mode == DGRAD) {
        const int t = kg / a.K, kout = kg - t * a.K;
        const int r = a.r0 + a.stride * (t / a.nq), q = a.q0 + a.stride * (t % a.nq);
        return to_f<T>(static_cast<const T*>(a.w)[((static_cast<int64_t>(kout) * a.R + r) * a.S + q) * a.C + j]);
    } else {
        const T* X = static_cast<const T*>(a.x);
        const int HoWo = a.Ho * a.Wo;
        const int m = kg;
        const int n = m / HoWo, rem = m - n * HoWo, oh = rem / a.Wo, ow = rem - oh * a.Wo;
        const int tap = j / a.C, c = j - tap * a.C, r = tap / a.S, q = tap - r * a.S;
        const int ih = oh * a.stride - a.pad + r, iw = ow * a.stride - a.pad + q;
        if (ih < 0 || ih >= a.H || iw < 0 || iw >= a.W) return 0.f;
        return to_f<T>(X[((static_cast<int64_t>(n) * a.H + ih) * a.W + iw) * a.C + c]);
    }
}

template <class T, int MODE>
__global__ void __launch_bounds__(256) conv_simt_kernel(ConvArgs a) {
    __shared__ float As[16][64 + 4];
    __shared__ float Bs[16][64 + 4];
    const int tid = threadIdx.x;
    const int m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
    const int tx = tid & 15, ty = tid >> 4;
    const int nkb_total = (a.KG + 15) / 16;
    int kb0 = 0, kb1 = nkb_total;
    if (MODE == WGRAD) {
        kb0 = blockIdx.z * a.kb_per_split;
        kb1 = min(nkb_total, kb0 + a.kb_per_split);
    }
    float acc[4][4] = {};
    for (int kb = kb0; kb < kb1; ++kb) {
        for (int e = tid; e < 16 * 64; e += 256) {
            const int kk = e / 64, mm = e % 64;
            As[kk][mm] = a_elem<T>(a, MODE, m0 + mm, kb * 16 + kk);
            Bs[kk][mm] = b_elem<T>(a, MODE, n0 + mm, kb * 16 + kk);
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += av[i] * bv[j];
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty * 4 + i;
        if (m >= a.M) continue;
        int64_t row;
        if (MODE == FPROP) {
            row = static_cast<int64_t>(m) * a.NG;
        } else if (MODE == DGRAD) {
            const int HpWp = a.Hp * a.Wp;
            const int n = m / HpWp, rem = m - n * HpWp, i2 = rem / a.Wp, j2 = rem - i2 * a.Wp;
            row = ((static_cast<int64_t>(n) * a.H + a.ph + a.stride * i2) * a.W + a.pw + a.stride * j2) * a.C;
        } else {
            row = (static_cast<int64_t>(blockIdx.z) * a.M + m) * a.NG;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n >= a.NG) continue;
            if (MODE == WGRAD) {
                static_cast<float*>(a.out)[row + n] = acc[i][j];
            } else {
                T* o = static_cast<T*>(a.out) + row + n;
                float f = acc[i][j];
                if (MODE == DGRAD && a.accumulate) f += to_f<T>(static_cast<const T*>(a.addend)[o - static_cast<T*>(a.out)]);
                if (MODE == DGRAD && a.mask) {
                    f = to_f<T>(from_f<T>(f));
                    if (!(to_f<T>(static_cast<const T*>(a.mask)[o - static_cast<T*>(a.out)]) > 0.f))
                        f = __fmul_rn(a.mask_neg, f);
                }
                *o = from_f<T>(f);
            }
        }
    }
}

// deterministic split-K reduction: dw[i] = sum_s ws[s][i] (fixed order), cast
template <class T>
__global__ void wgrad_reduce_kernel(const float* __restrict__ ws, int splits, int64_t n, T* __restrict__ dw) {
    pdl_wait();
    pdl_trigger();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float s = 0.f;
        int k = 0;
        for (; k + 4 <= splits; k += 4) {
            const float a0 = ws[k * n + i], a1 = ws[(k + 1) * n + i], a2 = ws[(k + 2) * n + i], a3 = ws[(k + 3) * n + i];
            s += a0;
            s += a1;
            s += a2;
            s += a3;
        }
        for (; k < splits; ++k) s += ws[k * n + i];
        dw[i] = from_f<T>(s);
    }
}

// same, from transposed partials ws[s][j][i] (j < n_rows = R*S*C, i < n_cols = K)
// into dw[i][j]: 32x32 tiles through shared memory, both sides coalesced
template <class T>
__global__ void wgrad_reduce_t_kernel(const float* __restrict__ ws, int splits, int n_rows, int n_cols,
                                      T* __restrict__ dw) {
    __shared__ float tile[32][33];
    pdl_wait();
    pdl_trigger();
    const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    const int64_t per = static_cast<int64_t>(n_rows) * n_cols;
    // 4 rows per thread, the split loop unrolled by 4: 16 independent loads in
    // flight per thread (a dependent load chain per split was latency-bound)
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const int i = i0 + tx;
    bool ok[4];
    int64_t off[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int j = j0 + ty + 8 * u;
        ok[u] = j < n_rows && i < n_cols;
        off[u] = ok[u] ? static_cast<int64_t>(j) * n_cols + i : 0;
    }
    int k = 0;
    for (; k + 4 <= splits; k += 4) {
        float v[4][4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int u = 0; u < 4; ++u) v[kk][u] = ok[u] ? ws[(k + kk) * per + off[u]] : 0.f;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] += v[kk][u];
    }
    for (; k < splits; ++k)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += ok[u] ? ws[k * per + off[u]] : 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) tile[ty + 8 * u][tx] = acc[u];
    __syncthreads();
    for (int ii = ty; ii < 32; ii += 8) {
        const int i = i0 + ii, j = j0 + tx;
        if (i < n_cols && j < n_rows) dw[static_cast<int64_t>(i) * n_rows + j] = from_f<T>(tile[tx][ii]);
    }
}

// All deferred split-K reductions of a backward pass in one launch: CTA b
// finds its job in the tile prefix table, then reduces one 32x32 tile exactly
// like wgrad_reduce_t_kernel (transposed jobs) or wgrad_reduce_kernel (plain
// [K][RSC] partials) -- same per-element summation order (splits in order).
// binary16 bits with an all-ones exponent: inf or NaN
SDB_DEV bool h_nonfinite(__half h) { return (__half_as_ushort(h) & 0x7c00u) == 0x7c00u; }

__global__ void __launch_bounds__(256) wgrad_reduce_batched_kernel(const WgradJob* __restrict__ jobs,
                                                                  const int* __restrict__ tile_start, int njobs,
                                                                  int* __restrict__ nonfinite) {
    // has_nonfinite (src/trainer.cpp:78-82) of the fp16 gradients this launch
    // writes, OR-ed into *nonfinite: the optimizer needs no separate pass
    __shared__ float tile[32][33];
    pdl_wait();
    pdl_trigger();
    bool bad = false;
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tile_start[mid] <= static_cast<int>(blockIdx.x)) lo = mid;
        else hi = mid - 1;
    }
    const WgradJob jb = jobs[lo];
    const int t = blockIdx.x - tile_start[lo];
    const int tiles_j = (jb.rows + 31) / 32;
    const int j0 = (t % tiles_j) * 32, i0 = (t / tiles_j) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t per = static_cast<int64_t>(jb.rows) * jb.cols;
    // element (j, i) of partial s at ws[s][j][i]: rows j (R*S*C for transposed jobs, K otherwise)
    if ((jb.cols & 3) == 0) {
        // vector path: thread = (row j, 4 consecutive columns), one 16-byte load
        // per split; same fixed split order, so bit-identical to the scalar path
        const int q = threadIdx.x & 7, jr = threadIdx.x >> 3;
        const int j = j0 + jr, iq = i0 + 4 * q;
        const bool okv = j < jb.rows && iq < jb.cols;
        const float4* src = reinterpret_cast<const float4*>(jb.ws + (okv ? static_cast<int64_t>(j) * jb.cols + iq : 0));
        const int64_t per4 = per / 4;
        float4 a4 = make_float4(0.f, 0.f, 0.f, 0.f);
        int k = 0;
        for (; k + 4 <= jb.splits; k += 4) {
            float4 v[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) v[kk] = okv ? src[(k + kk) * per4] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                a4.x += v[kk].x;
                a4.y += v[kk].y;
                a4.z += v[kk].z;
                a4.w += v[kk].w;
            }
        }
        for (; k < jb.splits; ++k) {
            const float4 v = okv ? src[k * per4] : make_float4(0.f, 0.f, 0.f, 0.f);
            a4.x += v.x;
            a4.y += v.y;
            a4.z += v.z;
            a4.w += v.w;
        }
        __half* dw = static_cast<__half*>(jb.dw);
        if (jb.transposed) {
            tile[jr][4 * q] = a4.x;
            tile[jr][4 * q + 1] = a4.y;
            tile[jr][4 * q + 2] = a4.z;
            tile[jr][4 * q + 3] = a4.w;
            __syncthreads();
            for (int ii = ty; ii < 32; ii += 8) {
                const int io = i0 + ii, jo = j0 + tx;
                if (io < jb.cols && jo < jb.rows) {
                    const __half hv = __float2half_rn(tile[tx][ii]);
                    bad |= h_nonfinite(hv);
                    dw[static_cast<int64_t>(io) * jb.rows + jo] = hv;
                }
            }
        } else if (okv) {
            __half2* o = reinterpret_cast<__half2*>(dw + static_cast<int64_t>(j) * jb.cols + iq);
            const __half2 h0 = __floats2half2_rn(a4.x, a4.y), h1 = __floats2half2_rn(a4.z, a4.w);
            bad |= h_nonfinite(__low2half(h0)) | h_nonfinite(__high2half(h0)) | h_nonfinite(__low2half(h1)) |
                   h_nonfinite(__high2half(h1));
            o[0] = h0;
            o[1] = h1;
        }
        if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
        return;
    }
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const int i = i0 + tx;
    bool ok[4];
    int64_t off[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int j = j0 + ty + 8 * u;
        ok[u] = j < jb.rows && i < jb.cols;
        off[u] = ok[u] ? static_cast<int64_t>(j) * jb.cols + i : 0;
    }
    int k = 0;
    for (; k + 4 <= jb.splits; k += 4) {
        float v[4][4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int u = 0; u < 4; ++u) v[kk][u] = ok[u] ? jb.ws[(k + kk) * per + off[u]] : 0.f;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] += v[kk][u];
    }
    for (; k < jb.splits; ++k)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += ok[u] ? jb.ws[k * per + off[u]] : 0.f;
    __half* dw = static_cast<__half*>(jb.dw);
    if (jb.transposed) {
#pragma unroll
        for (int u = 0; u < 4; ++u) tile[ty + 8 * u][tx] = acc[u];
        __syncthreads();
        for (int ii = ty; ii < 32; ii += 8) {
            const int io = i0 + ii, jo = j0 + tx;
            if (io < jb.cols && jo < jb.rows) {
                const __half hv = __float2half_rn(tile[tx][ii]);
                bad |= h_nonfinite(hv);
                dw[static_cast<int64_t>(io) * jb.rows + jo] = hv;
            }
        }
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (ok[u]) {
                const __half hv = __float2half_rn(acc[u]);
                bad |= h_nonfinite(hv);
                dw[off[u]] = hv;
            }
    }
    if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
}

cudaError_t wgrad_reduce_batched(const WgradJob* jobs_dev, const int* tile_start_dev, int njobs, int total_tiles,
                                 cudaStream_t st, int* nonfinite) {
    if (njobs == 0) return cudaSuccess;
    return launch_pdl(wgrad_reduce_batched_kernel, dim3(total_tiles), dim3(256), 0, st, jobs_dev, tile_start_dev, njobs,
                      nonfinite);
}

int wgrad_job_tiles(const WgradJob& j) { return ((j.rows + 31) / 32) * ((j.cols + 31) / 32); }

// zero the dgrad output positions of a phase with no taps
template <class T>
__global__ void dgrad_zero_phase_kernel(ConvArgs a) {
    const int64_t total = static_cast<int64_t>(a.M) * a.C;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int m = static_cast<int>(e / a.C), c = static_cast<int>(e % a.C);
        const int HpWp = a.Hp * a.Wp;
        const int n = m / HpWp, rem = m - n * HpWp, i2 = rem / a.Wp, j2 = rem - i2 * a.Wp;
        T* o = static_cast<T*>(a.out) +
               ((static_cast<int64_t>(n) * a.H + a.ph + a.stride * i2) * a.W + a.pw + a.stride * j2) * a.C + c;
        if (!a.accumulate) *o = from_f<T>(0.f);
    }
}

// ============================================================ launchers
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool make_tmap(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                      const uint32_t* box, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn), cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return false;
    }
    cuuint64_t d[5], st[4];
    cuuint32_t b[5], es[5];
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
        es[i] = 1;
        if (i + 1 < rank) st[i] = strides[i];
    }
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rank, const_cast<void*>(base), d, st, b, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// cuTensorMapEncodeIm2col: 4-D NHWC tensor [N][H][W][C] fp16, SWIZZLE_128B,
// 64 channels per pixel (128 B rows), `pixels` output pixels per box
typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

static bool make_im2col(CUtensorMap* m, const void* base, int N, int H, int W, int C, int lower_h, int lower_w,
                        int upper_h, int upper_w, int stride, int pixels) {
    static EncodeIm2colFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", reinterpret_cast<void**>(&fn), cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return false;
    }
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                                static_cast<cuuint64_t>(N)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(C) * 2, static_cast<cuuint64_t>(W) * C * 2,
                                   static_cast<cuuint64_t>(H) * W * C * 2};
    const int lower[2] = {lower_w, lower_h};
    const int upper[2] = {upper_w, upper_h};
    const cuuint32_t es[4] = {1, static_cast<cuuint32_t>(stride), static_cast<cuuint32_t>(stride), 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(base), dims, strides, lower, upper, 64,
              static_cast<cuuint32_t>(pixels), es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool& tma_disabled_flag() {
    static bool f = std::getenv("SDB_CONV_NO_TMA") != nullptr;
    return f;
}

// all-TMA path applicability (see conv_tma_kernel)
static bool tma_ok(const ConvArgs& a, int mode) {
    if (tma_disabled_flag()) return false;
    if (mode == DGRAD) return (a.K % kBK) == 0;
    return (a.C % 64) == 0;
}

template <int MODE, int BN, int ST, int EPI = 0, int EW = (BN == 256 ? 8 : 4)>
static cudaError_t launch_tma(ConvArgs a, int splits, cudaStream_t st, ConvStats* cst = nullptr) {
    using Cfg = TmaCfg<MODE, BN, ST, EPI, EW>;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(conv_tma_kernel<MODE, BN, ST, EPI, EW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg::kSmem);
        configured = true;
    }
    const int tiles_m = (a.M + kBM - 1) / kBM, tiles_n = (a.NG + BN - 1) / BN;
    const int n_tiles = tiles_m * tiles_n * splits;
    int grid = std::min(n_tiles, Cfg::kPerSM * kNumSMs);
    // fused output statistics need every CTA on one column block (grid a
    // multiple of tiles_n): e.g. the res5 expansion convs (tiles_n = 8) give up
    // 4 of 148 CTAs (< 3% of a ~80 us GEMM) to save a 50 us statistics pass
    if (((MODE == FPROP && EPI == 0) || EPI == 2) && cst && grid % tiles_n != 0 && grid >= tiles_n)
        grid -= grid % tiles_n;
    if (MODE == WGRAD) {
        // experiment knob: SMs a wgrad may occupy (leaves room for the concurrent norm chain)
        static const int cap = [] { const char* e = std::getenv("SDB_WGRAD_SMS"); return e ? std::atoi(e) : 0; }();
        if (cap > 0) grid = std::min(grid, Cfg::kPerSM * cap);
    }
    TmaPair tm;
    std::memset(&tm, 0, sizeof(tm));
    bool ok;
    a.plain = (a.R == 1 && a.S == 1 && a.stride == 1 && a.pad == 0) ? 1 : 0;
    // plain 2-D view of the activation operand: [pixels][channels]
    auto plain_map = [&](CUtensorMap* m, const void* p, int64_t pixels, int chans, uint32_t box_pixels) {
        const uint64_t dims[2] = {static_cast<uint64_t>(chans), static_cast<uint64_t>(pixels)};
        const uint64_t strides[1] = {static_cast<uint64_t>(chans) * 2};
        const uint32_t box[2] = {64, box_pixels};
        return make_tmap(m, p, 2, dims, strides, box);
    };
    if (MODE == FPROP) {
        ok = a.plain ? plain_map(&tm.a, a.x, static_cast<int64_t>(a.N) * a.H * a.W, a.C, kBM)
                     : make_im2col(&tm.a, a.x, a.N, a.H, a.W, a.C, -a.pad, -a.pad, a.pad - (a.R - 1),
                                   a.pad - (a.S - 1), a.stride, kBM);
        const uint64_t dims[2] = {static_cast<uint64_t>(a.KG), static_cast<uint64_t>(a.NG)};
        const uint64_t strides[1] = {static_cast<uint64_t>(a.KG) * 2};
        const uint32_t box[2] = {64, static_cast<uint32_t>(BN)};
        ok = ok && make_tmap(&tm.b, a.w, 2, dims, strides, box);
    } else if (MODE == DGRAD) {
        // DY over the phase grid: Hp x Wp output positions, base shifted by (nr-1, nq-1)
        const int lh = (a.ph + a.pad - a.r0) / a.stride - (a.nr - 1);
        const int lw = (a.pw + a.pad - a.q0) / a.stride - (a.nq - 1);
        ok = a.plain ? plain_map(&tm.a, a.x, static_cast<int64_t>(a.N) * a.Ho * a.Wo, a.K, kBM)
                     : make_im2col(&tm.a, a.x, a.N, a.Ho, a.Wo, a.K, lh, lw, a.Hp - a.Ho + lh, a.Wp - a.Wo + lw, 1, kBM);
        const uint64_t dims[3] = {static_cast<uint64_t>(a.C), static_cast<uint64_t>(a.R) * a.S, static_cast<uint64_t>(a.K)};
        const uint64_t strides[2] = {static_cast<uint64_t>(a.C) * 2, static_cast<uint64_t>(a.R) * a.S * a.C * 2};
        const uint32_t box[3] = {64, 1, 64};
        ok = ok && make_tmap(&tm.b, a.w, 3, dims, strides, box);
    } else {
        // transposed orientation: M = (r,s,c), N = k; DY viewed as [pixels][k]
        ok = a.plain ? plain_map(&tm.a, a.x, static_cast<int64_t>(a.N) * a.H * a.W, a.C, kBK)
                     : make_im2col(&tm.a, a.x, a.N, a.H, a.W, a.C, -a.pad, -a.pad, a.pad - (a.R - 1),
                                   a.pad - (a.S - 1), a.stride, kBK);
        const uint64_t dims[2] = {static_cast<uint64_t>(a.NG), static_cast<uint64_t>(a.KG)};
        const uint64_t strides[1] = {static_cast<uint64_t>(a.NG) * 2};
        const uint32_t box[2] = {64, 64};
        ok = ok && make_tmap(&tm.b, a.w, 2, dims, strides, box);
    }
    // fp16 output through TMA stores: fprop, and stride-1 dgrad without the
    // residual addend / activation mask (SDB_CONV_NO_TMA_STORE disables).  It
    // pays where the epilogue bounds the tile (short K: <= 4 k-blocks) or the
    // mainloop is long enough to hide it (3x3); for 1x1 convs with 8+ k-blocks
    // the stores compete with the operand loads for the TMA unit (measured
    // 1.1x slower on the res5 expansion convs), so those keep the LSU stores.
    static const bool no_tma_store = std::getenv("SDB_CONV_NO_TMA_STORE") != nullptr;
    a.tma_out = 0;
    const bool epi_pays = a.R * a.S > 1 || (a.KG + kBK - 1) / kBK <= 4;
    // an fprop whose output statistics are wanted always takes the TMA-store
    // epilogue: the fused statistics save a full read pass of the output,
    // more than the slower stores cost on 8+ k-block 1x1 shapes
    static const bool stats_force = std::getenv("SDB_STATS_NO_FORCE_TMA") == nullptr;
    if (ok && !no_tma_store && (epi_pays || (MODE == FPROP && cst && stats_force)) &&
        (MODE == FPROP || (MODE == DGRAD && a.stride == 1 && !a.accumulate && !a.mask))) {
        const int cols = MODE == FPROP ? a.NG : a.C;
        const int64_t rows = MODE == FPROP ? static_cast<int64_t>(a.M) : static_cast<int64_t>(a.N) * a.H * a.W;
        if ((cols % 8) == 0) {
            const uint64_t dims[2] = {static_cast<uint64_t>(cols), static_cast<uint64_t>(rows)};
            const uint64_t strides[1] = {static_cast<uint64_t>(cols) * 2};
            const uint32_t box[2] = {static_cast<uint32_t>(Cfg::kSC), 32};
            a.tma_out = make_tmap(&tm.o, a.out, 2, dims, strides, box,
                                  Cfg::kSC == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B)
                            ? 1
                            : 0;
        }
    }
    if (EPI == 1 && ok) {
        // output and residual addend views [N*H*W][C], 32 x 32 boxes
        const uint64_t dims[2] = {static_cast<uint64_t>(a.C), static_cast<uint64_t>(a.N) * a.H * a.W};
        const uint64_t strides[1] = {static_cast<uint64_t>(a.C) * 2};
        const uint32_t box[2] = {static_cast<uint32_t>(Cfg::kSC), 32};
        ok = make_tmap(&tm.o, a.out, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B) &&
             make_tmap(&tm.r, a.addend, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B);
        a.tma_out = 0;
    }
    if (EPI == 2 && ok) {
        // output and stored-y views [N*H*W][C], SC x 32 boxes (the IABN-backward statistics)
        const uint64_t dims[2] = {static_cast<uint64_t>(a.C), static_cast<uint64_t>(a.N) * a.H * a.W};
        const uint64_t strides[1] = {static_cast<uint64_t>(a.C) * 2};
        const uint32_t box[2] = {static_cast<uint32_t>(Cfg::kSC), 32};
        const CUtensorMapSwizzle swz = Cfg::kSC == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
        ok = cst && cst->bs_y && make_tmap(&tm.o, a.out, 2, dims, strides, box, swz) &&
             make_tmap(&tm.r, cst->bs_y, 2, dims, strides, box, swz);
        a.tma_out = 0;
        if (ok) {
            const size_t need = static_cast<size_t>(grid) * 4 * 2 * BN * sizeof(double);
            if (grid % tiles_n != 0 || need > cst->cap_bytes) return cudaErrorInvalidValue;
            a.stats = cst->buf;
            cst->produced = 1;
            cst->ctas = grid;
            cst->tiles_n = tiles_n;
            cst->bn = BN;
        }
        if (!ok) return cudaErrorInvalidValue;
        return launch_pdl(conv_tma_kernel<MODE, BN, ST, EPI, EW>, dim3(grid), dim3(Cfg::kThreads), Cfg::kSmem, st, a,
                          tiles_m, tiles_n, n_tiles, tm);
    }
    if (!ok) return cudaErrorInvalidValue;
    a.stats = nullptr;
    if (cst) {
        cst->produced = 0;
        static const bool no_fused_stats = std::getenv("SDB_NO_FUSED_STATS") != nullptr;
        const size_t need = static_cast<size_t>(grid) * 4 * 2 * BN * sizeof(double);
        if (MODE == FPROP && EPI == 0 && a.tma_out && splits == 1 && grid % tiles_n == 0 && need <= cst->cap_bytes &&
            !no_fused_stats) {
            a.stats = cst->buf;
            cst->produced = 1;
            cst->ctas = grid;
            cst->tiles_n = tiles_n;
            cst->bn = BN;
        }
    }
    return launch_pdl(conv_tma_kernel<MODE, BN, ST, EPI, EW>, dim3(grid), dim3(Cfg::kThreads), Cfg::kSmem, st, a, tiles_m,
                      tiles_n, n_tiles, tm);
}

// tile width: 256 when the GEMM N is wide enough (one CTA per SM, 2 x 256 TMEM
// columns), else 128 / 64 (two CTAs per SM)
// fprop/dgrad: when 128x256 tiles would leave more than half of the 148 SMs
// idle (small-M res4 layers with N = 256: 66 tiles), 128x64 tiles (264, two
// CTAs per SM) -- these one-tile-per-CTA layers are latency-bound, not
// L2-bound: two independent tile pipelines per SM hide each other's fill and
// drain (ncu: 128x128 -> 128x64 0.78x on the fprops, 0.71x on the dgrads with
// fused statistics; SDB_CONV_NARROW128 restores 128).  wgrad fills the machine
// with split-K instead.
static int tma_bn(const ConvArgs& a, int mode = WGRAD) {
    if (a.NG >= 256) {
        const int64_t tiles256 = static_cast<int64_t>((a.M + kBM - 1) / kBM) * ((a.NG + 255) / 256);
        static const bool no_narrow = std::getenv("SDB_CONV_NO_NARROW") != nullptr;
        static const bool bn128 = std::getenv("SDB_CONV_NARROW128") != nullptr;
        if (mode != WGRAD && 2 * tiles256 <= kNumSMs && !no_narrow) return bn128 ? 128 : 64;
        return 256;
    }
    return a.NG > 64 ? 128 : 64;
}

template <int MODE>
static cudaError_t launch_tma_pick(const ConvArgs& a, int splits, cudaStream_t st, ConvStats* cst = nullptr) {
    switch (tma_bn(a, MODE)) {
        case 256: {
            // fprop with fused norm statistics and a short reduction (<= 16 k-blocks):
            // the epilogue is the longer half of the tile pipeline -> 16 epilogue warps
            // (3 stages fit beside their staging; the res5 1x1 512 -> 2048 fprop with
            // statistics 130 -> 121 us; at 32 k-blocks the 4th stage matters more)
            static const bool ew16 = std::getenv("SDB_NO_EPI16") == nullptr;
            if (MODE == FPROP && cst && ew16 && a.KG <= 16 * kBK)
                return launch_tma<MODE, 256, 3, 0, 16>(a, splits, st, cst);
            return launch_tma<MODE, 256, 4>(a, splits, st, cst);
        }
        case 128: return launch_tma<MODE, 128, 3>(a, splits, st, cst);
        default: return launch_tma<MODE, 64, 4>(a, splits, st, cst);
    }
}

template <int MODE, int BN, int ST>
static cudaError_t launch_tc(const ConvArgs& a, int splits, cudaStream_t st) {
    using Cfg = TcPCfg<MODE, BN, ST>;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(conv_tc_kernel<MODE, BN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
        configured = true;
    }
    const int tiles_m = (a.M + kBM - 1) / kBM, tiles_n = (a.NG + BN - 1) / BN;
    const int n_tiles = tiles_m * tiles_n * splits;
    // resident CTAs per SM: TMEM holds 512 columns (2 accumulators of BN each) and
    // 227 KB of shared memory
    const int per_sm = (4 * BN <= 512 && 2 * (Cfg::kSmem + 1024) <= 228 * 1024) ? 2 : 1;
    const int grid = std::min(n_tiles, per_sm * kNumSMs);
    TmaDesc tma;
    std::memset(&tma, 0, sizeof(tma));
    bool ok = true;
    if (MODE == FPROP) {
        // filter [K][R*S*C] fp16, box [BN rows][64 k]
        const uint64_t dims[2] = {static_cast<uint64_t>(a.KG), static_cast<uint64_t>(a.NG)};
        const uint64_t strides[1] = {static_cast<uint64_t>(a.KG) * 2};
        const uint32_t box[2] = {64, static_cast<uint32_t>(BN)};
        ok = make_tmap(&tma.m, a.w, 2, dims, strides, box);
    } else if (MODE == DGRAD && a.tma_b) {
        // filter [K][R*S][C] fp16, box [64 kout][1 tap][64 c]
        const uint64_t dims[3] = {static_cast<uint64_t>(a.C), static_cast<uint64_t>(a.R) * a.S, static_cast<uint64_t>(a.K)};
        const uint64_t strides[2] = {static_cast<uint64_t>(a.C) * 2, static_cast<uint64_t>(a.R) * a.S * a.C * 2};
        const uint32_t box[3] = {64, 1, 64};
        ok = make_tmap(&tma.m, a.w, 3, dims, strides, box);
    } else if (MODE == WGRAD) {
        // DY [pixels][K] fp16, box [64 pixels][64 kout]
        const uint64_t dims[2] = {static_cast<uint64_t>(a.M), static_cast<uint64_t>(a.KG)};
        const uint64_t strides[1] = {static_cast<uint64_t>(a.M) * 2};
        const uint32_t box[2] = {64, 64};
        ok = make_tmap(&tma.m, a.w, 2, dims, strides, box);
    }
    if (!ok) return cudaErrorInvalidValue;
    conv_tc_kernel<MODE, BN, ST><<<grid, Cfg::kThreads, Cfg::kSmem, st>>>(a, tiles_m, tiles_n, n_tiles, tma);
    return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_tc_pick(const ConvArgs& a, int splits, cudaStream_t st) {
    if (a.NG <= 64) return launch_tc<MODE, 64, 4>(a, splits, st);
    const int64_t tiles128 = static_cast<int64_t>((a.M + 127) / 128) * ((a.NG + 127) / 128) * splits;
    if (a.NG >= 256 && tiles128 >= 2 * kNumSMs) return launch_tc<MODE, 256, 4>(a, splits, st);
    return launch_tc<MODE, 128, 3>(a, splits, st);
}

template <class T, int MODE>
static cudaError_t launch_simt(const ConvArgs& a, int splits, cudaStream_t st) {
    dim3 grid((a.M + 63) / 64, (a.NG + 63) / 64, splits);
    conv_simt_kernel<T, MODE><<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

static ConvArgs make_args(const ConvShape& g) {
    ConvArgs a{};
    a.N = g.N; a.H = g.H; a.W = g.W; a.C = g.C; a.K = g.K; a.R = g.R; a.S = g.S;
    a.stride = g.stride; a.pad = g.pad;
    a.Ho = (g.H + 2 * g.pad - g.R) / g.stride + 1;
    a.Wo = (g.W + 2 * g.pad - g.S) / g.stride + 1;
    return a;
}

static bool tc_ok(const ConvShape& g, int dtype) {
    return dtype == kF16 && (g.C % 8) == 0 && (g.K % 8) == 0 && !conv_force_simt();
}

static bool& force_simt_flag() {
    static bool f = false;
    return f;
}
bool conv_force_simt() { return force_simt_flag(); }
void conv_set_force_simt(bool v) { force_simt_flag() = v; }

cudaError_t conv_fprop(const ConvShape& g, int dtype, const void* x, const void* w, void* y, cudaStream_t st,
                       ConvStats* cst) {
    ConvArgs a = make_args(g);
    a.x = x; a.w = w; a.out = y;
    a.M = g.N * a.Ho * a.Wo;
    a.NG = g.K;
    a.KG = g.R * g.S * g.C;
    if (cst) cst->produced = 0;
    if (tc_ok(g, dtype))
        return tma_ok(a, FPROP) ? launch_tma_pick<FPROP>(a, 1, st, cst) : launch_tc_pick<FPROP>(a, 1, st);
    return dtype == kF16 ? launch_simt<__half, FPROP>(a, 1, st) : launch_simt<float, FPROP>(a, 1, st);
}

cudaError_t conv_dgrad(const ConvShape& g, int dtype, const void* dy, const void* w, void* dx, int accumulate,
                       cudaStream_t st, const void* addend, const void* mask, float mask_neg,
                       const uint8_t* mask_bits, ConvStats* bstats) {
    ConvArgs base = make_args(g);
    base.x = dy; base.w = w; base.out = dx; base.accumulate = accumulate || addend != nullptr;
    base.mask = mask;
    base.mbits = mask_bits;
    base.mask_neg = mask_neg;
    base.addend = addend ? addend : dx;
    base.NG = g.C;
    const int sd = g.stride;
    // phases whose taps are all empty (e.g. the odd pixels of a 1x1 stride-2
    // conv) receive no gradient: zero the whole output once with a contiguous
    // memset (or leave it untouched when accumulating)
    if (mask && tc_ok(g, dtype) && (g.K % kBK) != 0) return cudaErrorNotSupported;  // mask: TMA / SIMT epilogues only
    bool empty_phase = false;
    for (int ph = 0; ph < sd; ++ph)
        for (int pw = 0; pw < sd; ++pw) {
            const int r0 = (ph + g.pad) % sd, q0 = (pw + g.pad) % sd;
            if (r0 >= g.R || q0 >= g.S) empty_phase = true;
        }
    // positions no tap reaches keep the addend (or zero) unmasked: only valid
    // when they are zero, i.e. without a separate addend
    if (mask && empty_phase && base.accumulate && base.addend != dx) return cudaErrorNotSupported;
    if (empty_phase && base.accumulate && base.addend != dx) {
        // taps never reach some output phases: those positions take the addend as is
        const cudaError_t e = cudaMemcpyAsync(dx, base.addend,
                                              static_cast<size_t>(g.N) * g.H * g.W * g.C * (dtype == kF16 ? 2 : 4),
                                              cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
        base.addend = dx;
    }
    if (empty_phase && !base.accumulate) {
        const cudaError_t e = cudaMemsetAsync(dx, 0, static_cast<size_t>(g.N) * g.H * g.W * g.C * (dtype == kF16 ? 2 : 4), st);
        if (e != cudaSuccess) return e;
    }
    for (int ph = 0; ph < sd; ++ph)
        for (int pw = 0; pw < sd; ++pw) {
            ConvArgs a = base;
            a.ph = ph; a.pw = pw;
            a.Hp = ph < g.H ? (g.H - ph + sd - 1) / sd : 0;
            a.Wp = pw < g.W ? (g.W - pw + sd - 1) / sd : 0;
            if (a.Hp == 0 || a.Wp == 0) continue;
            a.r0 = (ph + g.pad) % sd;
            a.q0 = (pw + g.pad) % sd;
            a.nr = a.r0 < g.R ? (g.R - a.r0 + sd - 1) / sd : 0;
            a.nq = a.q0 < g.S ? (g.S - a.q0 + sd - 1) / sd : 0;
            a.M = g.N * a.Hp * a.Wp;
            a.KG = a.nr * a.nq * g.K;
            cudaError_t e;
            if (a.KG == 0) {
                continue;  // zeroed above (or untouched when accumulating)
            } else if (tc_ok(g, dtype)) {
                a.tma_b = (g.K % kBK) == 0 ? 1 : 0;
                static const bool no_resid = std::getenv("SDB_CONV_NO_RESID_EPI") != nullptr;
                static const bool no_bstats = std::getenv("SDB_NO_FUSED_BWD_STATS") != nullptr;
                if (bstats) bstats->produced = 0;
                if (bstats && bstats->bs_y && !no_bstats && tma_ok(a, DGRAD) && sd == 1 && !a.accumulate && !a.mask &&
                    (g.C % 16) == 0 && tma_bn(a, DGRAD) <= 128) {
                    a.bs_gamma = bstats->bs_gamma;
                    a.bs_beta = bstats->bs_beta;
                    a.bs_slope = bstats->bs_slope;
                    // BN <= 128 only: the 256-wide tile cannot keep its 4 mainloop stages
                    // next to the y ring, and 3 stages cost the res5 dgrads more than
                    // the statistics pass they save (measured)
                    if (tma_bn(a, DGRAD) == 128) e = launch_tma<DGRAD, 128, 3, 2>(a, 1, st, bstats);
                    else e = launch_tma<DGRAD, 64, 4, 2>(a, 1, st, bstats);
                } else if (tma_ok(a, DGRAD) && a.mbits && a.accumulate && sd == 1 && tma_bn(a, DGRAD) == 256 &&
                           (g.C % 32) == 0 && !no_resid)
                    e = launch_tma<DGRAD, 256, 3, 1>(a, 1, st);
                else
                    e = tma_ok(a, DGRAD) ? launch_tma_pick<DGRAD>(a, 1, st) : launch_tc_pick<DGRAD>(a, 1, st);
            } else {
                e = dtype == kF16 ? launch_simt<__half, DGRAD>(a, 1, st) : launch_simt<float, DGRAD>(a, 1, st);
            }
            if (e != cudaSuccess) return e;
        }
    return cudaSuccess;
}

// Deterministic split-K plan for wgrad (shared by workspace sizing and launch):
// fill one wave of the tensor-core kernel (1 CTA/SM at BN=256, 2 at BN<=128)
// with >= 8 k-blocks per split.
static int wgrad_splits(const ConvShape& g, int dtype) {
    ConvArgs a = make_args(g);
    a.M = g.K;
    a.NG = g.R * g.S * g.C;
    a.KG = g.N * a.Ho * a.Wo;
    const int64_t M = a.M, NG = a.NG, KG = a.KG;
    const bool tc = tc_ok(g, dtype);
    const int bk = tc ? kBK : 16;
    const int64_t nkb = (KG + bk - 1) / bk;
    int64_t tiles, per_sm;
    if (tc && tma_ok(a, WGRAD)) {
        // transposed orientation: GEMM M = R*S*C, N = K
        std::swap(a.M, a.NG);
        const int bn = tma_bn(a);
        tiles = ((a.M + 127) / 128) * ((a.NG + bn - 1) / bn);
        per_sm = bn <= 128 ? 2 : 1;
    } else if (tc) {
        const int bn = NG <= 64 ? 64 : 128;  // split-K launches never pick BN=256 unless tiles are plentiful
        tiles = ((M + 127) / 128) * ((NG + bn - 1) / bn);
        per_sm = 2;
    } else {
        tiles = ((M + 63) / 64) * ((NG + 63) / 64);
        per_sm = 4;
    }
    const int64_t target = per_sm * kNumSMs;
    int64_t splits = target / std::max<int64_t>(tiles, 1);
    // every split writes a full fp32 partial tile (which the reduce reads back):
    // keep each split at least kMinKb k-blocks long so that partial traffic
    // stays well below the operand traffic.  Measured on the C4 step (CUDA
    // graph, wgrads on the side stream): 8 -> 13.06 ms, 24 -> 11.73,
    // 32 -> 11.62, 48 -> 11.99 (785 MB -> ~300 MB of partials per step, and
    // wgrad grids that leave SMs to the concurrent dgrad/norm chain)
    static const int64_t kMinKb = [] {
        const char* e = std::getenv("SDB_WGRAD_MINKB");
        return e ? std::max(1, std::atoi(e)) : 32;
    }();
    splits = std::max<int64_t>(1, std::min<int64_t>(splits, nkb / kMinKb));
    return static_cast<int>(std::min<int64_t>(splits, 64));
}

size_t conv_wgrad_workspace(const ConvShape& g, int dtype) {
    const int64_t M = g.K, NG = static_cast<int64_t>(g.R) * g.S * g.C;
    return static_cast<size_t>(wgrad_splits(g, dtype)) * M * NG * sizeof(float);
}

cudaError_t conv_wgrad(const ConvShape& g, int dtype, const void* x, const void* dy, void* dw, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
    return conv_wgrad_deferred(g, dtype, x, dy, dw, ws, ws_bytes, st, nullptr);
}

cudaError_t conv_wgrad_deferred(const ConvShape& g, int dtype, const void* x, const void* dy, void* dw, void* ws,
                                size_t ws_bytes, cudaStream_t st, WgradJob* job) {
    ConvArgs a = make_args(g);
    a.x = x; a.w = dy;
    a.M = g.K;
    a.NG = g.R * g.S * g.C;
    a.KG = g.N * a.Ho * a.Wo;
    const bool tc = tc_ok(g, dtype);
    const int bk = tc ? kBK : 16;
    const int nkb = (a.KG + bk - 1) / bk;
    const int64_t per = static_cast<int64_t>(a.M) * a.NG;
    int splits = wgrad_splits(g, dtype);
    a.kb_per_split = (nkb + splits - 1) / splits;
    splits = (nkb + a.kb_per_split - 1) / a.kb_per_split;
    if (ws == nullptr || ws_bytes < static_cast<size_t>(per) * sizeof(float) * splits) return cudaErrorInvalidValue;
    a.out = ws;
    cudaError_t e;
    if (tc && tma_ok(a, WGRAD)) {
        ConvArgs at = a;
        std::swap(at.M, at.NG);  // partials [split][(r,s,c)][k]
        // diagnostic only (wrong gradients): time the step without the wgrad GEMMs
        static const bool skip = std::getenv("SDB_DIAG_SKIP_WGRAD") != nullptr;
        e = skip && job ? cudaSuccess : launch_tma_pick<WGRAD>(at, splits, st);
        if (e != cudaSuccess) return e;
        if (job) {
            *job = WgradJob{static_cast<const float*>(ws), dw, splits, at.M, at.NG, 1};
            return cudaSuccess;
        }
        const dim3 grid((at.M + 31) / 32, (at.NG + 31) / 32);
        if (dtype == kF16)
            return launch_pdl(wgrad_reduce_t_kernel<__half>, grid, dim3(256), 0, st, static_cast<const float*>(ws),
                              splits, at.M, at.NG, static_cast<__half*>(dw));
        return launch_pdl(wgrad_reduce_t_kernel<float>, grid, dim3(256), 0, st, static_cast<const float*>(ws), splits,
                          at.M, at.NG, static_cast<float*>(dw));
    }
    if (tc) e = launch_tc_pick<WGRAD>(a, splits, st);
    else e = dtype == kF16 ? launch_simt<__half, WGRAD>(a, splits, st) : launch_simt<float, WGRAD>(a, splits, st);
    if (e != cudaSuccess) return e;
    if (job) {
        *job = WgradJob{static_cast<const float*>(ws), dw, splits, a.M, a.NG, 0};
        return cudaSuccess;
    }
    const int blocks = static_cast<int>(std::min<int64_t>((per + 255) / 256, 8 * kNumSMs));
    if (dtype == kF16)
        return launch_pdl(wgrad_reduce_kernel<__half>, dim3(blocks), dim3(256), 0, st, static_cast<const float*>(ws),
                          splits, per, static_cast<__half*>(dw));
    return launch_pdl(wgrad_reduce_kernel<float>, dim3(blocks), dim3(256), 0, st, static_cast<const float*>(ws), splits,
                      per, static_cast<float*>(dw));
}

}  // namespace sdb
