// roi.cu -- RoIAlign forward/backward, pooling, residual activations, detection
// losses and the synthetic input generator.
//
// RoIAlign: aligned (half-pixel) corners, fixed sampling ratio, average of the
// bilinear samples; the restated oracle is orc_roialign_fwd/bwd (numerically
// identical to torchvision.ops.roi_align(aligned=True)).  Forward: one warp
// per (RoI, bin row, 256 channels), lane = 8 channels, coalesced 512-byte
// corner-row reads through L1 (below).
// Backward is a deterministic GATHER (no atomics): one warp per (pixel,
// channel slab) walks the RoIs whose nonzero-weight box holds its pixel in
// index order and accumulates, from the separable per-RoI weight tables
// WY[h][ph] x WX[w][pw], every dY contribution in a fixed order -- bitwise
// reproducible run to run.
//
// Losses fold the loss scale into backward exactly like the reference CE op
// (src/model.cpp:132-150): forward returns the unscaled loss, backward
// multiplies by grad_scale.  Reductions are fixed-order (deterministic).
// Compiled with -fmad=false (no contraction) so float expressions evaluate
// as written in the oracle.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "detect.h"
#include "sdb_internal.h"

namespace sdb {

namespace {

template <class T>
SDB_DEV void ld8(const T* p, float (&v)[8]);
template <>
SDB_DEV void ld8<__half>(const __half* p, float (&v)[8]) {
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
SDB_DEV void ld8<float>(const float* p, float (&v)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <class T>
SDB_DEV void st8(T* p, const float (&v)[8]);
template <>
SDB_DEV void st8<__half>(__half* p, const float (&v)[8]) {
    uint4 u;
    __half2* h = reinterpret_cast<__half2*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = u;
}
template <>
SDB_DEV void st8<float>(float* p, const float (&v)[8]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}

// 8 channels as 4 fp32 pairs (packed-FMA operands)
template <class T>
SDB_DEV void ld8x2(const T* p, float2 (&v)[4]);
template <>
SDB_DEV void ld8x2<__half>(const __half* p, float2 (&v)[4]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __half22float2(h[i]);
}
template <>
SDB_DEV void ld8x2<float>(const float* p, float2 (&v)[4]) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = make_float2(a.x, a.y); v[1] = make_float2(a.z, a.w); v[2] = make_float2(b.x, b.y); v[3] = make_float2(b.z, b.w);
}
template <class T>
SDB_DEV void st8x2(T* p, const float2 (&v)[4]) {
    float f[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) { f[2 * i] = v[i].x; f[2 * i + 1] = v[i].y; }
    st8<T>(p, f);
}

struct Geom {
    int b;
    float sw, sh, bw, bh;
};

// orc roi_geom (aligned=1): corner * scale - 0.5, bins = extent / P
SDB_DEV Geom roi_geom(const float* r, int P, float scale) {
    Geom g;
    g.b = static_cast<int>(r[0]);
    g.sw = r[1] * scale - 0.5f;
    g.sh = r[2] * scale - 0.5f;
    const float ew = r[3] * scale - 0.5f, eh = r[4] * scale - 0.5f;
    g.bw = (ew - g.sw) / static_cast<float>(P);
    g.bh = (eh - g.sh) / static_cast<float>(P);
    return g;
}

SDB_DEV float sample_coord(float start, int p, float bin, int i, int sr) {
    return start + static_cast<float>(p) * bin + (static_cast<float>(i) + 0.5f) * bin / static_cast<float>(sr);
}

// ---------------------------------------------------------------- RoIAlign fwd
template <class T>
__global__ void roialign_fwd_kernel(const T* __restrict__ feat, int H, int W, int C, const float* __restrict__ rois,
                                    int R, int P, float scale, int sr, int step, T* __restrict__ out) {
    // output bins: every `step`-th bin of the P x P grid (Po x Po of them)
    const int C8 = C / 8;
    const int Po = (P + step - 1) / step;
    const int64_t total = static_cast<int64_t>(R) * Po * Po * C8;
    const float count = static_cast<float>(max(sr * sr, 1));
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c8 = static_cast<int>(e % C8);
        const int64_t bin = e / C8;
        const int pw = static_cast<int>(bin % Po) * step, ph = static_cast<int>((bin / Po) % Po) * step;
        const int r = static_cast<int>(bin / (Po * Po));
        const Geom g = roi_geom(rois + static_cast<int64_t>(r) * 5, P, scale);
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (g.b >= 0) {
            const T* f = feat + static_cast<int64_t>(g.b) * H * W * C + c8 * 8;
            for (int iy = 0; iy < sr; ++iy) {
                float y = sample_coord(g.sh, ph, g.bh, iy, sr);
                for (int ix = 0; ix < sr; ++ix) {
                    float x = sample_coord(g.sw, pw, g.bw, ix, sr);
                    if (y < -1.0f || y > static_cast<float>(H) || x < -1.0f || x > static_cast<float>(W)) continue;
                    float yy = y <= 0.f ? 0.f : y, xx = x <= 0.f ? 0.f : x;
                    int yl = static_cast<int>(yy), xl = static_cast<int>(xx), yh, xh;
                    if (yl >= H - 1) { yh = yl = H - 1; yy = static_cast<float>(yl); } else yh = yl + 1;
                    if (xl >= W - 1) { xh = xl = W - 1; xx = static_cast<float>(xl); } else xh = xl + 1;
                    const float ly = yy - static_cast<float>(yl), lx = xx - static_cast<float>(xl);
                    const float hy = 1.f - ly, hx = 1.f - lx;
                    const float w1 = hy * hx, w2 = hy * lx, w3 = ly * hx, w4 = ly * lx;
                    float v1[8], v2[8], v3[8], v4[8];
                    ld8<T>(f + (static_cast<int64_t>(yl) * W + xl) * C, v1);
                    ld8<T>(f + (static_cast<int64_t>(yl) * W + xh) * C, v2);
                    ld8<T>(f + (static_cast<int64_t>(yh) * W + xl) * C, v3);
                    ld8<T>(f + (static_cast<int64_t>(yh) * W + xh) * C, v4);
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j] += w1 * v1[j] + w2 * v2[j] + w3 * v3[j] + w4 * v4[j];
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = acc[j] / count;
        }
        st8<T>(out + e * 8, acc);
    }
}

// ---------------------------------------------------------------- RoIAlign fwd (smem-staged)
// One CTA per (image, 8-channel slab): the slab of the image's whole feature
// map is staged in shared memory once (16 B per pixel in fp16), so the 16
// bilinear corner reads of every output bin
// hit smem instead of L2 (the RoIs of an image overlap heavily: at C4 every
// feature pixel is read by ~100 RoI samples; through L2 that read
// amplification capped the direct kernel at ~1.6 GB of L2 traffic per step).
// The image's RoIs are taken in chunks of kRaChunk: the separable sample
// table of a chunk -- per (RoI, axis, bin, sample): element offsets of the
// low/high pixel row (y) or column (x) and their bilinear weights, zero
// weights for samples outside [-1, H] -- is built once in smem, then every
// (RoI, bin) item of the chunk reads it and blends its 16 corners with packed
// fp32 FMAs (fma.rn.f32x2).  Same sample positions, clamps and corner weights
// as the direct kernel above.
constexpr int kRaChunk = 32;
constexpr int kRaFwdThreads = 512;

struct RaTab {
    int lo, hi;  // element offsets into the staged slab (row * W * 8 for y, col * 8 for x)
    float wl, wh;
};

SDB_DEV RaTab ra_axis(float v, int lim, int mult) {
    RaTab t{0, 0, 0.f, 0.f};
    if (v < -1.0f || v > static_cast<float>(lim)) return t;
    if (v <= 0.f) v = 0.f;
    int lo = static_cast<int>(v), hi;
    if (lo >= lim - 1) { hi = lo = lim - 1; v = static_cast<float>(lo); } else hi = lo + 1;
    t.lo = lo * mult;
    t.hi = hi * mult;
    t.wh = v - static_cast<float>(lo);
    t.wl = 1.f - t.wh;
    return t;
}

// one bin: the SR x SR samples' 16 corners blended with packed fp32 FMAs
// (compile-time SR: all corner loads of the bin are issued back to back)
template <class T, int SR>
SDB_DEV void ra_bin(const T* f, const RaTab* ty, const RaTab* tx, int sr, float2 (&acc)[4]) {
    const int n = SR > 0 ? SR : sr;
#pragma unroll
    for (int iy = 0; iy < (SR > 0 ? SR : 1); ++iy) {
        for (int iy2 = iy; iy2 < (SR > 0 ? iy + 1 : n); ++iy2) {
            const RaTab Y = ty[iy2];
#pragma unroll
            for (int ix = 0; ix < (SR > 0 ? SR : 1); ++ix) {
                for (int ix2 = ix; ix2 < (SR > 0 ? ix + 1 : n); ++ix2) {
                    const RaTab X = tx[ix2];
                    const float2 w1 = make_float2(Y.wl * X.wl, Y.wl * X.wl), w2 = make_float2(Y.wl * X.wh, Y.wl * X.wh);
                    const float2 w3 = make_float2(Y.wh * X.wl, Y.wh * X.wl), w4 = make_float2(Y.wh * X.wh, Y.wh * X.wh);
                    float2 v1[4], v2[4], v3[4], v4[4];
                    ld8x2<T>(f + Y.lo + X.lo, v1);
                    ld8x2<T>(f + Y.lo + X.hi, v2);
                    ld8x2<T>(f + Y.hi + X.lo, v3);
                    ld8x2<T>(f + Y.hi + X.hi, v4);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        acc[k] = ffma2(w4, v4[k], ffma2(w3, v3[k], ffma2(w2, v2[k], ffma2(w1, v1[k], acc[k]))));
                }
            }
        }
    }
}

template <class T, int SR>
__global__ void __launch_bounds__(kRaFwdThreads) roialign_fwd_smem_kernel(const T* __restrict__ feat, int H, int W,
                                                                          int C, const float* __restrict__ rois, int R,
                                                                          int P, float scale, int sr, int step,
                                                                          T* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char ra_smem[];
    const int n = blockIdx.y, c8 = blockIdx.x;
    const int HW = H * W;
    const int Po = (P + step - 1) / step, PP = Po * Po;
    T* fs = reinterpret_cast<T*>(ra_smem);  // [HW][8]
    int* list = reinterpret_cast<int*>(ra_smem + static_cast<size_t>(HW) * 8 * sizeof(T));
    RaTab* tab = reinterpret_cast<RaTab*>(list + ((R + 3) & ~3));  // [kRaChunk][2][Po][sr]
    __shared__ int cnt;
    if (threadIdx.x == 0) cnt = 0;
    const T* src = feat + static_cast<int64_t>(n) * HW * C + c8 * 8;
    for (int p = threadIdx.x; p < HW; p += blockDim.x) {
        const uint4* s = reinterpret_cast<const uint4*>(src + static_cast<int64_t>(p) * C);
        uint4* d = reinterpret_cast<uint4*>(fs + static_cast<size_t>(p) * 8);
        d[0] = __ldg(s);
        if (sizeof(T) == 4) d[1] = __ldg(s + 1);
    }
    __syncthreads();
    // this image's RoIs (order irrelevant: every output bin is written by one thread)
    for (int r = threadIdx.x; r < R; r += blockDim.x)
        if (static_cast<int>(rois[static_cast<int64_t>(r) * 5]) == n) list[atomicAdd(&cnt, 1)] = r;
    __syncthreads();
    const int total = cnt;
    const float inv_count = 1.0f / static_cast<float>(max(sr * sr, 1));
    const float2 ic = make_float2(inv_count, inv_count);
    const int per_roi = 2 * Po * sr;
    for (int r0 = 0; r0 < total; r0 += kRaChunk) {
        const int nr = min(kRaChunk, total - r0);
        for (int t = threadIdx.x; t < nr * per_roi; t += blockDim.x) {
            const int j = t / per_roi, q = t - j * per_roi;
            const int axis = q / (Po * sr), q2 = q - axis * Po * sr;
            const int pb = q2 / sr, is = q2 - pb * sr;
            const Geom g = roi_geom(rois + static_cast<int64_t>(list[r0 + j]) * 5, P, scale);
            tab[t] = axis ? ra_axis(sample_coord(g.sw, pb * step, g.bw, is, sr), W, 8)
                          : ra_axis(sample_coord(g.sh, pb * step, g.bh, is, sr), H, W * 8);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < nr * PP; e += blockDim.x) {
            const int j = e / PP, bin = e - j * PP;
            const int ph = bin / Po, pw = bin - ph * Po;
            float2 acc[4] = {};
            ra_bin<T, SR>(fs, tab + j * per_roi + ph * sr, tab + j * per_roi + Po * sr + pw * sr, sr, acc);
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] = ffma2(acc[k], ic, make_float2(0.f, 0.f));
            st8x2<T>(out + (static_cast<int64_t>(list[r0 + j]) * PP + bin) * C + c8 * 8, acc);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- RoIAlign bwd
// dX[n, y, x, c] = sum over RoIs r of image n (index order), bins (ph, pw)
// (row-major) of WY_r[y][ph] * WX_r[x][pw] / sr^2 * dY[r, ph, pw, c], with
// WY_r[y][ph] = the bilinear weights of pixel row y summed over the samples of
// bin row ph (separable).  A deterministic GATHER, no atomics:
//   1. roialign_bwd_weights_kernel: one warp per RoI tabulates WY_r / WX_r for
//      every pixel row / column and the bounding box of the nonzero ones
//      (shared by all pixels and channel slabs: computed once per step);
//   2. roialign_tile_list_kernel / roialign_seg_plan_kernel: per 4x4 pixel
//      block, the RoIs that reach it (index order) and their exact pair
//      count, cut into work-balanced segments (below);
//   3. roialign_bwd_gather_kernel: one CTA per (block, segment), one warp per
//      (pixel, 256*V-channel slab), lane = V 8-channel chunks; it walks the
//      segment's RoIs whose box holds its pixel (ballot, list order), fetches
//      the RoI's 2 x pw weights of its row and column in one load per lane,
//      and accumulates the nonzero bin pairs in registers; the dY rows the
//      block's pixels share hit L1.
// The summation order per output element is fixed (segment, RoI, ph, pw) --
// bitwise reproducible run to run; products are accumulated with packed fp32
// FMAs.
constexpr int kRaBlk = 4;  // CTA = kRaBlk x kRaBlk pixels (one warp each)

SDB_DEV float bin_axis_weight(float start, float bin, int pb_full, int sr, int pix, int lim) {
    float wsum = 0.f;
    for (int is = 0; is < sr; ++is) {
        float v = sample_coord(start, pb_full, bin, is, sr);
        if (v < -1.0f || v > static_cast<float>(lim)) continue;
        if (v <= 0.f) v = 0.f;
        int lo_i = static_cast<int>(v), hi_i;
        if (lo_i >= lim - 1) { hi_i = lo_i = lim - 1; v = static_cast<float>(lo_i); } else hi_i = lo_i + 1;
        const float l = v - static_cast<float>(lo_i), h = 1.f - l;
        if (lo_i == pix) wsum += h;
        if (hi_i == pix) wsum += l;
    }
    return wsum;
}

__global__ void __launch_bounds__(256) roialign_bwd_weights_kernel(const float* __restrict__ rois, int R, int H, int W,
                                                                   int P, float scale, int sr, int step, int pw,
                                                                   float* __restrict__ tab, int4* __restrict__ box,
                                                                   uint8_t* __restrict__ nzc) {
    const int r = static_cast<int>((blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= R) return;
    const Geom g = roi_geom(rois + static_cast<int64_t>(r) * 5, P, scale);
    const int Po = (P + step - 1) / step;
    float* ty = tab + static_cast<int64_t>(r) * (H + W) * pw;
    int ylo = 0x7fff, yhi = -1, xlo = 0x7fff, xhi = -1;
    for (int t = lane; t < H + W; t += 32) {
        const bool isx = t >= H;
        const int pix = isx ? t - H : t;
        bool any = false;
        int nz = 0;
        for (int pb = 0; pb < pw; ++pb) {
            const float w = pb < Po ? (isx ? bin_axis_weight(g.sw, g.bw, pb * step, sr, pix, W)
                                           : bin_axis_weight(g.sh, g.bh, pb * step, sr, pix, H))
                                    : 0.f;
            ty[static_cast<int64_t>(t) * pw + pb] = w;
            any |= w != 0.f;
            nz += w != 0.f;
        }
        nzc[static_cast<int64_t>(r) * (H + W) + t] = static_cast<uint8_t>(nz);
        if (any) {
            if (isx) { xlo = min(xlo, pix); xhi = max(xhi, pix); }
            else { ylo = min(ylo, pix); yhi = max(yhi, pix); }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ylo = min(ylo, __shfl_xor_sync(0xffffffffu, ylo, o));
        yhi = max(yhi, __shfl_xor_sync(0xffffffffu, yhi, o));
        xlo = min(xlo, __shfl_xor_sync(0xffffffffu, xlo, o));
        xhi = max(xhi, __shfl_xor_sync(0xffffffffu, xhi, o));
    }
    if (lane == 0) {
        const bool empty = yhi < 0 || xhi < 0 || g.b < 0;
        box[r] = make_int4(empty ? -1 : g.b, ylo | (max(yhi, 0) << 16), xlo | (max(xhi, 0) << 16), 0);
    }
}

// Work balance.  The gather above walks, per pixel warp, every RoI that
// reaches its pixel: where the trained RPN stacks hundreds of small RoIs on a
// few pixels (thousands of (RoI, bin) contributions on one pixel), that one
// warp's serial walk was the whole kernel's duration (0.68-2.9 ms instead of
// 0.14-0.2).  So the pixel blocks' RoI lists are built once
// (roialign_tile_list_kernel, index order), each block's work -- its exact
// (pixel, RoI, bin) pair count, from per-row / per-column nonzero-bin counts
// of the weight table -- is cut into up to kRaSegMax consecutive segments of
// about kRaSegWork pairs, and one CTA takes each segment: a single-segment
// block writes dX directly; a split block's segments write fp32 partials and
// the last to finish (ticket) sums them in segment order.  Per element the
// order is fixed (segment, RoI, ph, pw): bitwise reproducible, no atomics on
// data.
constexpr int kRaSegMax = 32;
constexpr int kRaSegWork = 1024;  // (pixel, RoI, bin) pairs per segment at 7 x 7 bins, about
constexpr int kRaSlots = 512;     // partial-sum slots (segments of split blocks) per channel chunk

__global__ void __launch_bounds__(256) roialign_tile_list_kernel(const int4* __restrict__ box,
                                                                 const uint8_t* __restrict__ nzc, int R, int H, int W,
                                                                 long long seg_work, int* __restrict__ tl_cnt,
                                                                 int* __restrict__ tl_nseg,
                                                                 int* __restrict__ seg_start, int* __restrict__ tl) {
    extern __shared__ int wk[];  // [R] work of each listed RoI
    __shared__ int wsum[8];
    __shared__ long long wtot[8];
    __shared__ int cnt;
    __shared__ long long run;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int bxn = (W + kRaBlk - 1) / kRaBlk, byn = (H + kRaBlk - 1) / kRaBlk;
    const int tile = blockIdx.x, n = blockIdx.y;
    const int tx0 = (tile % bxn) * kRaBlk, ty0 = (tile / bxn) * kRaBlk;
    const int t = n * bxn * byn + tile;
    int* out = tl + static_cast<int64_t>(t) * R;
    if (tid == 0) cnt = 0;
    __syncthreads();
    for (int base = 0; base < R; base += 256) {
        bool hit = false;
        int w = 0;
        if (base + tid < R) {
            const int r = base + tid;
            const int4 b = __ldg(box + r);
            hit = b.x == n && (b.y & 0xffff) <= ty0 + kRaBlk - 1 && (b.y >> 16) >= ty0 &&
                  (b.z & 0xffff) <= tx0 + kRaBlk - 1 && (b.z >> 16) >= tx0;
            if (hit) {
                // pairs over the block's pixels: (sum of the rows' nonzero bins) x (columns')
                const uint8_t* c = nzc + static_cast<int64_t>(r) * (H + W);
                int a = 0, bb = 0;
                for (int k = 0; k < kRaBlk; ++k) {
                    if (ty0 + k < H) a += c[ty0 + k];
                    if (tx0 + k < W) bb += c[H + tx0 + k];
                }
                w = a * bb;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) wsum[warp] = __popc(m);
        __syncthreads();
        int off = cnt;
        for (int w2 = 0; w2 < warp; ++w2) off += wsum[w2];
        if (hit) {
            const int i = off + __popc(m & ((1u << lane) - 1u));
            out[i] = base + tid;
            wk[i] = w;
        }
        __syncthreads();
        if (tid == 0) {
            int s2 = 0;
            for (int w2 = 0; w2 < 8; ++w2) s2 += wsum[w2];
            cnt += s2;
        }
        __syncthreads();
    }
    const int nl = cnt;
    // total work -> segment count; cut where the running work passes s * total / ns
    long long my = 0;
    for (int i = tid; i < nl; i += 256) my += wk[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my += __shfl_xor_sync(0xffffffffu, my, o);
    if (lane == 0) wtot[warp] = my;
    __syncthreads();
    long long total = 0;
    for (int w2 = 0; w2 < 8; ++w2) total += wtot[w2];
    const long long nsl = (total + seg_work - 1) / seg_work;
    const int ns = nsl < 1 ? 1 : (nsl > kRaSegMax ? kRaSegMax : static_cast<int>(nsl));
    int* ss = seg_start + static_cast<int64_t>(t) * (kRaSegMax + 1);
    if (tid == 0) {
        tl_cnt[t] = nl;
        tl_nseg[t] = ns;
        ss[0] = 0;
        for (int s2 = 1; s2 <= ns; ++s2) ss[s2] = nl;  // segments left empty by heavy entries end at nl
        run = 0;
    }
    __syncthreads();
    if (ns > 1) {
        // entry i belongs to segment min(ns - 1, before_i * ns / total), before_i = the
        // work of the entries ahead of it (non-decreasing in i); a segment starts at its
        // first entry, one that no entry maps to is left empty
        for (int base = 0; base < nl; base += 256) {
            const int i = base + tid;
            const long long w = i < nl ? wk[i] : 0;
            long long v = w;  // inclusive warp scan
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long u = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += u;
            }
            if (lane == 31) wtot[warp] = v;
            __syncthreads();
            long long pre = run;
            for (int w2 = 0; w2 < warp; ++w2) pre += wtot[w2];
            const long long before = pre + v - w;
            if (i < nl) {
                const long long sq = (before * ns) / total;
                const int si = sq > ns - 1 ? ns - 1 : static_cast<int>(sq);
                if (si >= 1) atomicMin(&ss[si], i);
            }
            __syncthreads();
            if (tid == 0)
                for (int w2 = 0; w2 < 8; ++w2) run += wtot[w2];
            __syncthreads();
        }
        if (tid == 0)
            for (int s2 = ns - 1; s2 >= 1; --s2) ss[s2] = min(ss[s2], ss[s2 + 1]);
    }
}

// one CTA (block scans): the compact table of (block, segment) items and the
// partial slots of split blocks; a split whose slots would pass the capacity
// (counted over all requested splits ahead of it) keeps its block whole --
// slower, same sums
__global__ void __launch_bounds__(1024) roialign_seg_plan_kernel(const int* __restrict__ tl_nseg, int nt,
                                                                 int* __restrict__ seg, int* __restrict__ nseg_total,
                                                                 int* __restrict__ slot, unsigned* __restrict__ ticket,
                                                                 int nticket) {
    __shared__ int wa[32], wb[32];
    __shared__ int run_req, run_seg;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < nticket; i += blockDim.x) ticket[i] = 0u;
    if (tid == 0) run_req = run_seg = 0;
    __syncthreads();
    for (int base = 0; base < nt; base += 1024) {
        const int t = base + tid;
        const int req = t < nt ? tl_nseg[t] : 1;
        const int want = req > 1 ? req : 0;
        // exclusive prefix of the requested slots
        int a = want;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, a, o);
            if (lane >= o) a += u;
        }
        if (lane == 31) wa[warp] = a;
        __syncthreads();
        int pre = run_req;
        for (int w2 = 0; w2 < warp; ++w2) pre += wa[w2];
        const int before = pre + a - want;
        const bool split = want > 0 && before + want <= kRaSlots;
        const int ns = t < nt ? (split ? req : 1) : 0;
        // exclusive prefix of the segment items
        int b = ns;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, b, o);
            if (lane >= o) b += u;
        }
        if (lane == 31) wb[warp] = b;
        __syncthreads();
        int pre2 = run_seg;
        for (int w2 = 0; w2 < warp; ++w2) pre2 += wb[w2];
        const int k0 = pre2 + b - ns;
        if (t < nt) {
            slot[t] = split ? before : -1;
            for (int s2 = 0; s2 < ns; ++s2) seg[k0 + s2] = (t << 5) | s2;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w2 = 0; w2 < 32; ++w2) {
                run_req += wa[w2];
                run_seg += wb[w2];
            }
        }
        __syncthreads();
    }
    if (tid == 0) *nseg_total = run_seg;
}

// the per-pixel gather over one (block, segment) item at a time (persistent CTAs)
template <class T, int V>
__global__ void __launch_bounds__(kRaBlk * kRaBlk * 32) roialign_bwd_gather_kernel(
    const T* __restrict__ dy, int H, int W, int C, const int4* __restrict__ box, const float* __restrict__ tab, int R,
    int Po, int pw, float inv_count, T* __restrict__ dfeat, const int* __restrict__ tl_cnt,
    const int* __restrict__ tl_nseg, const int* __restrict__ seg_start, const int* __restrict__ tl,
    const int* __restrict__ seg, const int* __restrict__ nseg_total, const int* __restrict__ slot,
    unsigned* __restrict__ ticket, float* __restrict__ part) {
    __shared__ int s_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bxn = (W + kRaBlk - 1) / kRaBlk, byn = (H + kRaBlk - 1) / kRaBlk, ntiles = bxn * byn;
    const int chunk = blockIdx.y, nch = gridDim.y;
    const int c0 = chunk * 256 * V + lane * 8;
    const int64_t row_stride = static_cast<int64_t>(Po) * C;
    const int total = *nseg_total;
    for (int e = blockIdx.x; e < total; e += gridDim.x) {
        const int sv = seg[e], t = sv >> 5, sg = sv & 31;
        const int n = t / ntiles, tile = t - n * ntiles;
        const int y = (tile / bxn) * kRaBlk + warp / kRaBlk;
        const int x = (tile % bxn) * kRaBlk + warp % kRaBlk;
        const int sl = slot[t];
        const int ns = sl < 0 ? 1 : tl_nseg[t];
        const int* ss = seg_start + static_cast<int64_t>(t) * (kRaSegMax + 1);
        const int lo = sl < 0 ? 0 : ss[sg], hi = sl < 0 ? tl_cnt[t] : ss[sg + 1];
        const int* list = tl + static_cast<int64_t>(t) * R;
        const bool pix = y < H && x < W;
        float2 acc[V][4];
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[v][k] = make_float2(0.f, 0.f);
        if (pix) {
            for (int r0 = lo; r0 < hi; r0 += 32) {
                bool hit = false;
                int rl = 0;
                if (r0 + lane < hi) {
                    rl = __ldg(list + r0 + lane);
                    const int4 b = __ldg(box + rl);
                    hit = y >= (b.y & 0xffff) && y <= (b.y >> 16) && x >= (b.z & 0xffff) && x <= (b.z >> 16);
                }
                for (unsigned m = __ballot_sync(0xffffffffu, hit); m; m &= m - 1) {
                    const int r = __shfl_sync(0xffffffffu, rl, __ffs(m) - 1);
                    const float* trow = tab + static_cast<int64_t>(r) * (H + W) * pw;
                    float w = 0.f;
                    if (lane < pw) w = __ldg(trow + y * pw + lane);
                    else if (lane >= 16 && lane < 16 + pw) w = __ldg(trow + (H + x) * pw + (lane - 16));
                    const unsigned nz = __ballot_sync(0xffffffffu, w != 0.f);
                    const T* d = dy + static_cast<int64_t>(r) * Po * row_stride + c0;
                    for (unsigned a = nz & 0xffffu; a; a &= a - 1) {
                        const int ph = __ffs(a) - 1;
                        const float wy = __shfl_sync(0xffffffffu, w, ph);
                        for (unsigned b2 = nz >> 16; b2; b2 &= b2 - 1) {
                            const int pwi = __ffs(b2) - 1;
                            const float wx = __shfl_sync(0xffffffffu, w, 16 + pwi);
                            const float wgt = wy * wx * inv_count;
                            const float2 w2 = make_float2(wgt, wgt);
                            const T* dd = d + ph * row_stride + static_cast<int64_t>(pwi) * C;
#pragma unroll
                            for (int v = 0; v < V; ++v) {
                                if (c0 + v * 256 >= C) break;
                                float2 val[4];
                                ld8x2<T>(dd + v * 256, val);
#pragma unroll
                                for (int k = 0; k < 4; ++k) acc[v][k] = ffma2(w2, val[k], acc[v][k]);
                            }
                        }
                    }
                }
            }
        }
        if (ns == 1) {
            if (pix) {
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (c0 + v * 256 < C)
                        st8x2<T>(dfeat + ((static_cast<int64_t>(n) * H + y) * W + x) * C + c0 + v * 256, acc[v]);
            }
            continue;
        }
        // split block: this segment's partial; the last segment sums them in order
        const int64_t pstride = static_cast<int64_t>(kRaBlk * kRaBlk) * 256 * V;
        float* pp = part + (static_cast<int64_t>(sl + sg) * nch + chunk) * pstride + warp * 256 * V;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            float4* o = reinterpret_cast<float4*>(pp + v * 256 + lane * 8);
            o[0] = make_float4(acc[v][0].x, acc[v][0].y, acc[v][1].x, acc[v][1].y);
            o[1] = make_float4(acc[v][2].x, acc[v][2].y, acc[v][3].x, acc[v][3].y);
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(&ticket[t * nch + chunk], 1u) == static_cast<unsigned>(ns - 1);
        __syncthreads();
        if (!s_last) continue;
        __threadfence();
        if (threadIdx.x == 0) ticket[t * nch + chunk] = 0u;
        if (pix) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                if (c0 + v * 256 >= C) continue;
                float2 sum[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) sum[k] = make_float2(0.f, 0.f);
                for (int s2 = 0; s2 < ns; ++s2) {
                    const float4* q = reinterpret_cast<const float4*>(
                        part + (static_cast<int64_t>(sl + s2) * nch + chunk) * pstride + warp * 256 * V + v * 256 + lane * 8);
                    const float4 a0 = __ldcg(q), a1 = __ldcg(q + 1);
                    sum[0].x += a0.x; sum[0].y += a0.y; sum[1].x += a0.z; sum[1].y += a0.w;
                    sum[2].x += a1.x; sum[2].y += a1.y; sum[3].x += a1.z; sum[3].y += a1.w;
                }
                st8x2<T>(dfeat + ((static_cast<int64_t>(n) * H + y) * W + x) * C + c0 + v * 256, sum);
            }
        }
    }
}

// ---------------------------------------------------------------- RoIAlign fwd (warp per bin row)
// Lane = 8 channels of a 256-channel chunk, so every corner read is one
// coalesced 512-byte row piece through L1 (the image's feature map, 8.6 MB at
// C4, stays L2-resident; corners shared by neighbouring samples and bins hit
// L1).  A warp owns one (RoI, bin row, chunk): the bin row's sample rows are
// tabulated once, each bin's sample columns per bin, and the 4 corners of each
// sample are blended in the same order and with the same packed FMAs as the
// smem-staged kernel above (bit-identical outputs); every bin leaves as one
// coalesced 512-byte store.  (The smem-staged slab kernel is bound by shared-
// memory bank conflicts of its random per-thread corner reads -- 62 % of its
// wavefronts were conflicts in ncu -- and stays for sampling ratios != 2.)
constexpr int kRaWarps = 8;

template <class T, int SR>
__global__ void __launch_bounds__(32 * kRaWarps) roialign_fwd_warp_kernel(const T* __restrict__ feat, int H, int W,
                                                                           int C, const float* __restrict__ rois,
                                                                           int R, int P, float scale, int step,
                                                                           T* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int Po = (P + step - 1) / step;
    const int nch = (C + 255) / 256;
    const int gw = blockIdx.x * kRaWarps + (threadIdx.x >> 5);
    const int chunk = gw % nch, rest = gw / nch;
    const int phi = rest % Po, r = rest / Po;
    if (r >= R) return;
    const int c = chunk * 256 + lane * 8;
    if (c >= C) return;
    T* o = out + (static_cast<int64_t>(r) * Po + phi) * Po * C + c;
    const Geom g = roi_geom(rois + static_cast<int64_t>(r) * 5, P, scale);
    const float2 ic = make_float2(1.0f / (SR * SR), 1.0f / (SR * SR));
    if (g.b < 0) {
        const float2 z[4] = {};
        for (int pwi = 0; pwi < Po; ++pwi) st8x2<T>(o + static_cast<int64_t>(pwi) * C, z);
        return;
    }
    // element offsets (pixel row * W * C, pixel column * C) and weights
    RaTab ty[SR];
#pragma unroll
    for (int is = 0; is < SR; ++is) ty[is] = ra_axis(sample_coord(g.sh, phi * step, g.bh, is, SR), H, W * C);
    const T* f = feat + static_cast<int64_t>(g.b) * H * W * C + c;
    for (int pwi = 0; pwi < Po; ++pwi) {
        RaTab tx[SR];
#pragma unroll
        for (int is = 0; is < SR; ++is) tx[is] = ra_axis(sample_coord(g.sw, pwi * step, g.bw, is, SR), W, C);
        float2 acc[4] = {};
#pragma unroll
        for (int iy = 0; iy < SR; ++iy) {
            const RaTab Y = ty[iy];
            float2 v[SR][4][4];
#pragma unroll
            for (int ix = 0; ix < SR; ++ix) {
                const RaTab X = tx[ix];
                ld8x2<T>(f + Y.lo + X.lo, v[ix][0]);
                ld8x2<T>(f + Y.lo + X.hi, v[ix][1]);
                ld8x2<T>(f + Y.hi + X.lo, v[ix][2]);
                ld8x2<T>(f + Y.hi + X.hi, v[ix][3]);
            }
#pragma unroll
            for (int ix = 0; ix < SR; ++ix) {
                const RaTab X = tx[ix];
                const float2 w1 = make_float2(Y.wl * X.wl, Y.wl * X.wl), w2 = make_float2(Y.wl * X.wh, Y.wl * X.wh);
                const float2 w3 = make_float2(Y.wh * X.wl, Y.wh * X.wl), w4 = make_float2(Y.wh * X.wh, Y.wh * X.wh);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    acc[k] = ffma2(w4, v[ix][3][k], ffma2(w3, v[ix][2][k], ffma2(w2, v[ix][1][k], ffma2(w1, v[ix][0][k], acc[k]))));
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = ffma2(acc[k], ic, make_float2(0.f, 0.f));
        st8x2<T>(o + static_cast<int64_t>(pwi) * C, acc);
    }
}

// ---------------------------------------------------------------- pooling
// I = int32_t whenever the element count allows: the per-element index
// decomposition is then 32-bit (64-bit div/mod chains dominated these kernels)
template <class T, class I>
__global__ void maxpool_fwd_kernel(const T* __restrict__ x, int N, int H, int W, int C, int k, int s, int p,
                                   int Ho, int Wo, T* __restrict__ y, uint8_t* __restrict__ am) {
    const int C8 = C / 8;
    const I total = static_cast<I>(N) * Ho * Wo * C8;
    for (I e = blockIdx.x * static_cast<I>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<I>(gridDim.x) * blockDim.x) {
        const int c8 = static_cast<int>(e % C8);
        const I pix = e / C8;
        const int ow = static_cast<int>(pix % Wo), oh = static_cast<int>((pix / Wo) % Ho);
        const int n = static_cast<int>(pix / (static_cast<I>(Wo) * Ho));
        float m[8];
        int at[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) { m[j] = -INFINITY; at[j] = -1; }
        for (int r = 0; r < k; ++r)
            for (int q = 0; q < k; ++q) {
                const int ih = oh * s - p + r, iw = ow * s - p + q;
                if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
                float v[8];
                ld8<T>(x + ((static_cast<int64_t>(n) * H + ih) * W + iw) * C + c8 * 8, v);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (at[j] < 0 || v[j] > m[j]) { m[j] = v[j]; at[j] = r * k + q; }
            }
        st8<T>(y + static_cast<int64_t>(e) * 8, m);
        uint64_t pk = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) pk |= static_cast<uint64_t>(at[j] & 0xff) << (8 * j);
        reinterpret_cast<uint64_t*>(am)[e] = pk;
    }
}

// the stem pool forward (k 3, s 2, p 1): one CTA row per output row (n, oh),
// threads over (ow, 8-channel group) -- no per-element division chains; the
// same window order and tie rule as maxpool_fwd_kernel (first maximum in
// (r, q) order, padding taps skipped)
template <class T>
__global__ void __launch_bounds__(256) maxpool_fwd_k3s2_kernel(const T* __restrict__ x, int H, int W, int C8, int Ho,
                                                               int Wo, T* __restrict__ y, uint8_t* __restrict__ am) {
    const int orow = blockIdx.y;  // n * Ho + oh
    const int n = orow / Ho, oh = orow - n * Ho;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int ow = t / C8, c8 = t - ow * C8;
    if (ow >= Wo) return;
    float m[8];
    int at[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { m[j] = -INFINITY; at[j] = -1; }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const int ih = 2 * oh - 1 + r;
        if (ih < 0 || ih >= H) continue;
        const T* xr = x + (static_cast<int64_t>(n) * H + ih) * W * C8 * 8;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const int iw = 2 * ow - 1 + q;
            if (iw < 0 || iw >= W) continue;
            float v[8];
            ld8<T>(xr + (static_cast<int64_t>(iw) * C8 + c8) * 8, v);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (at[j] < 0 || v[j] > m[j]) { m[j] = v[j]; at[j] = r * 3 + q; }
        }
    }
    const int64_t e = (static_cast<int64_t>(orow) * Wo + ow) * C8 + c8;
    st8<T>(y + e * 8, m);
    uint64_t pk = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) pk |= static_cast<uint64_t>(at[j] & 0xff) << (8 * j);
    reinterpret_cast<uint64_t*>(am)[e] = pk;
}

template <class T, class I>
__global__ void maxpool_bwd_kernel(const T* __restrict__ dy, const uint8_t* __restrict__ am, int N, int H, int W, int C,
                                   int k, int s, int p, int Ho, int Wo, T* __restrict__ dx) {
    const int C8 = C / 8;
    const I total = static_cast<I>(N) * H * W * C8;
    for (I e = blockIdx.x * static_cast<I>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<I>(gridDim.x) * blockDim.x) {
        const int c8 = static_cast<int>(e % C8);
        const I pix = e / C8;
        const int iw = static_cast<int>(pix % W), ih = static_cast<int>((pix / W) % H);
        const int n = static_cast<int>(pix / (static_cast<I>(W) * H));
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int oh_lo = max(0, (ih + p - k + s) / s), oh_hi = min(Ho - 1, (ih + p) / s);
        const int ow_lo = max(0, (iw + p - k + s) / s), ow_hi = min(Wo - 1, (iw + p) / s);
        for (int oh = oh_lo; oh <= oh_hi; ++oh)
            for (int ow = ow_lo; ow <= ow_hi; ++ow) {
                const int r = ih - (oh * s - p), q = iw - (ow * s - p);
                if (r < 0 || r >= k || q < 0 || q >= k) continue;
                const int64_t oe = ((static_cast<int64_t>(n) * Ho + oh) * Wo + ow) * C8 + c8;
                const uint64_t pk = reinterpret_cast<const uint64_t*>(am)[oe];
                float g[8];
                ld8<T>(dy + oe * 8, g);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (static_cast<int>((pk >> (8 * j)) & 0xff) == r * k + q) acc[j] += g[j];
            }
        st8<T>(dx + static_cast<int64_t>(e) * 8, acc);
    }
}

// the ResNet stem pool (k 3, s 2, p 1): input row ih lies in window row ih/2
// (tap 1) when even, in window rows (ih-1)/2 (tap 2) and (ih+1)/2 (tap 0) when
// odd -- same for columns; one CTA row per input row, no division chains.
// Same window order (oh, ow ascending) and fp32 sums as the generic kernel.
template <class T>
__global__ void __launch_bounds__(256) maxpool_bwd_k3s2_kernel(const T* __restrict__ dy, const uint8_t* __restrict__ am,
                                                               int H, int W, int C8, int Ho, int Wo,
                                                               T* __restrict__ dx) {
    const int row = blockIdx.y;  // n * H + ih
    const int n = row / H, ih = row - n * H;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int iw = t / C8, c8 = t - iw * C8;
    if (iw >= W) return;
    int ohs[2], rs[2], nh = 0, ows[2], qs[2], nw = 0;
    if (ih & 1) {
        ohs[0] = (ih - 1) >> 1; rs[0] = 2;
        ohs[1] = (ih + 1) >> 1; rs[1] = 0;
        nh = ohs[1] < Ho ? 2 : 1;
    } else {
        ohs[0] = ih >> 1; rs[0] = 1; nh = ohs[0] < Ho ? 1 : 0;
    }
    if (iw & 1) {
        ows[0] = (iw - 1) >> 1; qs[0] = 2;
        ows[1] = (iw + 1) >> 1; qs[1] = 0;
        nw = ows[1] < Wo ? 2 : 1;
    } else {
        ows[0] = iw >> 1; qs[0] = 1; nw = ows[0] < Wo ? 1 : 0;
    }
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        if (a >= nh) break;
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            if (b >= nw) break;
            const int64_t oe = ((static_cast<int64_t>(n) * Ho + ohs[a]) * Wo + ows[b]) * C8 + c8;
            const uint64_t pk = __ldg(reinterpret_cast<const uint64_t*>(am) + oe);
            float g[8];
            ld8<T>(dy + oe * 8, g);
            const int tap = rs[a] * 3 + qs[b];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (static_cast<int>((pk >> (8 * j)) & 0xff) == tap) acc[j] += g[j];
        }
    }
    st8<T>(dx + ((static_cast<int64_t>(row) * W + iw) * C8 + c8) * 8, acc);
}

template <class T>
__global__ void avgpool_fwd_kernel(const T* __restrict__ x, int N, int HW, int C, T* __restrict__ y) {
    const int C8 = C / 8;
    const int64_t total = static_cast<int64_t>(N) * C8;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c8 = static_cast<int>(e % C8);
        const int64_t n = e / C8;
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int i = 0; i < HW; ++i) {
            float v[8];
            ld8<T>(x + (n * HW + i) * C + c8 * 8, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += v[j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = acc[j] / static_cast<float>(HW);
        st8<T>(y + e * 8, acc);
    }
}

// y (optional): the activation backward of the pooled tensor's producer fused
// in, exactly as the separate act_bwd pass on the rounded pooling gradient
template <class T, class I>
__global__ void avgpool_bwd_kernel(const T* __restrict__ dy, int N, int HW, int C, float inv, T* __restrict__ dx,
                                   const T* __restrict__ y, float neg, const uint8_t* __restrict__ ybits) {
    const int C8 = C / 8;
    const I total = static_cast<I>(N) * HW * C8;
    for (I e = blockIdx.x * static_cast<I>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<I>(gridDim.x) * blockDim.x) {
        const int c8 = static_cast<int>(e % C8);
        const I n = e / (static_cast<I>(HW) * C8);
        float g[8];
        ld8<T>(dy + (static_cast<int64_t>(n) * C8 + c8) * 8, g);
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = g[j] * inv;
        if (ybits) {
            // the activation's sign bitmap (bit j = y > 0) in place of y itself
            const unsigned int bm = ybits[e];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float r = to_f<T>(from_f<T>(g[j]));
                g[j] = ((bm >> j) & 1u) ? r : neg * r;
            }
        } else if (y) {
            float v[8];
            ld8<T>(y + static_cast<int64_t>(e) * 8, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float r = to_f<T>(from_f<T>(g[j]));
                g[j] = v[j] > 0.f ? r : neg * r;  // src/autograd.cpp:340-351
            }
        }
        st8<T>(dx + static_cast<int64_t>(e) * 8, g);
    }
}

// ---------------------------------------------------------------- elementwise
template <class T>
SDB_DEV float rnd(float v) {
    return to_f<T>(from_f<T>(v));
}

template <class T>
__global__ void add_act_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out, int64_t n8,
                               int act, float slope) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n8;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float va[8], vb[8], o[8];
        ld8<T>(a + e * 8, va);
        ld8<T>(b + e * 8, vb);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float s = rnd<T>(va[j] + vb[j]);  // add node output (src/tensor.cpp:125)
            o[j] = act == 0 ? s : (s > 0.f ? s : (act == 1 ? 0.f : slope * s));
        }
        st8<T>(out + e * 8, o);
    }
}

template <class T>
__global__ void act_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ y, T* __restrict__ dx, int64_t n8,
                               float neg) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n8;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float g[8], v[8];
        ld8<T>(dy + e * 8, g);
        ld8<T>(y + e * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = v[j] > 0.f ? g[j] : neg * g[j];  // src/autograd.cpp:340-351
        st8<T>(dx + e * 8, g);
    }
}

template <class T>
__global__ void relu_kernel(const T* __restrict__ x, T* __restrict__ y, int64_t n8) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n8;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float v[8];
        ld8<T>(x + e * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = v[j] > 0.f ? v[j] : 0.f;
        st8<T>(y + e * 8, v);
    }
}

template <class T>
__global__ void add_inplace_kernel(T* __restrict__ acc, const T* __restrict__ b, int64_t n8) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n8;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float va[8], vb[8];
        ld8<T>(acc + e * 8, va);
        ld8<T>(b + e * 8, vb);
#pragma unroll
        for (int j = 0; j < 8; ++j) va[j] += vb[j];
        st8<T>(acc + e * 8, va);
    }
}

// ---------------------------------------------------------------- losses
constexpr int kLossThreads = 1024;

SDB_DEV double block_sum_d(double v, double* sh) {
    v = warp_sum(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += sh[w];
    __syncthreads();
    return t;
}

template <class T>
SDB_DEV float ldv(const T* p, int64_t i) { return to_f<T>(p[i]); }

// reference softmax-CE (src/model.cpp:106-150) over rows with label >= 0
template <class T>
__global__ void __launch_bounds__(kLossThreads) softmax_ce_kernel(const T* __restrict__ logits, int R, int ncls, int ld,
                                                                  const int32_t* __restrict__ labels,
                                                                  T* __restrict__ dlogits, const double* scale,
                                                                  double* loss_out, int slot) {
    __shared__ double sh[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int cnt = 0;
    for (int r = threadIdx.x; r < R; r += blockDim.x) cnt += labels[r] >= 0;
    const double B = block_sum_d(static_cast<double>(cnt), sh);
    const double gs = scale ? *scale : 1.0;
    const float g = B > 0 ? static_cast<float>(1.0 * gs / B) : 0.f;
    double wl = 0.0;
    for (int r = wid; r < R; r += nw) {
        const int y = labels[r];
        const T* x = logits + static_cast<int64_t>(r) * ld;
        T* dx = dlogits + static_cast<int64_t>(r) * ld;
        if (y < 0) {
            for (int j = lane; j < ld; j += 32) dx[j] = from_f<T>(0.f);
            continue;
        }
        double mx = -INFINITY;
        for (int j = lane; j < ncls; j += 32) mx = fmax(mx, static_cast<double>(ldv(x, j)));
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        double z = 0.0;
        for (int j = lane; j < ncls; j += 32) z += exp(static_cast<double>(ldv(x, j)) - mx);
        z = warp_sum(z);
        float py = 0.f;
        for (int j = lane; j < ld; j += 32) {
            if (j < ncls) {
                const float pj = static_cast<float>(exp(static_cast<double>(ldv(x, j)) - mx) / z);
                if (j == y) py = pj;
                dx[j] = from_f<T>((pj - (j == y ? 1.0f : 0.0f)) * g);
            } else {
                dx[j] = from_f<T>(0.f);
            }
        }
        py = __shfl_sync(0xffffffffu, py, y & 31);
        if (lane == 0) wl += -log(fmax(1e-30, static_cast<double>(py)));
    }
    if (lane == 0) sh[wid] = wl;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t += sh[w];
        loss_out[slot] = B > 0 ? t / B : 0.0;
    }
}

// RPN losses run on many blocks with fixed-order partial sums (deterministic):
// per-block partials -> one tiny in-order reduction.
constexpr int kLossBlocks = 2 * kNumSMs;
constexpr int kLossBlockThreads = 256;

SDB_DEV double block_sum_d256(double v, double* sh) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < kLossBlockThreads / 32; ++w) t += sh[w];
    __syncthreads();
    return t;
}

// number of sampled anchors (label >= 0) per block
__global__ void __launch_bounds__(kLossBlockThreads) label_count_kernel(const int8_t* __restrict__ labels, int64_t n,
                                                                        double* __restrict__ partial) {
    __shared__ double sh[8];
    double c = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        c += labels[i] >= 0;
    const double t = block_sum_d256(c, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

SDB_DEV double sum_partials(const double* p, int n) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += p[i];
    return t;
}

// sigmoid BCE over anchors with label >= 0, normalised by their count
template <class T>
__global__ void __launch_bounds__(kLossBlockThreads) sigmoid_bce_kernel(const T* __restrict__ logits, int64_t n_loc,
                                                                        int A, int A_pad,
                                                                        const int8_t* __restrict__ labels,
                                                                        T* __restrict__ dlogits, const double* scale,
                                                                        const double* __restrict__ counts,
                                                                        double* __restrict__ partial) {
    __shared__ double sh[8];
    __shared__ double norm_s;
    if (threadIdx.x == 0) norm_s = sum_partials(counts, gridDim.x);
    __syncthreads();
    const double norm = norm_s;
    const double gs = (scale ? *scale : 1.0) / (norm > 0 ? norm : 1.0);
    const int64_t n = n_loc * A_pad;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int a = static_cast<int>(i % A_pad);
        float gout = 0.f;
        if (a < A) {
            const int t = labels[(i / A_pad) * A + a];
            if (t >= 0) {
                const double v = ldv(logits, i);
                acc += fmax(v, 0.0) - v * t + log1p(exp(-fabs(v)));
                gout = static_cast<float>((1.0 / (1.0 + exp(-v)) - t) * gs);
            }
        }
        dlogits[i] = from_f<T>(gout);
    }
    const double tot = block_sum_d256(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// loss = sum(partial) / (norm or sum(counts))
__global__ void loss_finalize_kernel(const double* __restrict__ partial, int n, const double* __restrict__ counts,
                                     double norm, double* loss_out, int slot) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double d = counts ? sum_partials(counts, n) : norm;
    const double t = sum_partials(partial, n);
    loss_out[slot] = d > 0 ? t / d : 0.0;
}

SDB_DEV void sl1(double d, double beta, double& l, double& g) {
    const double ad = fabs(d);
    if (ad < beta) {
        l = 0.5 * d * d / beta;
        g = d / beta;
    } else {
        l = ad - 0.5 * beta;
        g = d > 0 ? 1.0 : -1.0;
    }
}

// Multi-CTA variants (the single-CTA kernels above took ~100 us each at
// R = 1024): every CTA recounts the valid rows (R labels, a few KB), handles 8
// rows (one warp per row for CE) and writes a per-row / per-CTA fp64 loss; a
// one-warp kernel then sums them in a fixed order (deterministic).
constexpr int kRowsPerCta = 8;

template <class T>
__global__ void __launch_bounds__(256) softmax_ce_mc_kernel(const T* __restrict__ logits, int R, int ncls, int ld,
                                                            const int32_t* __restrict__ labels,
                                                            T* __restrict__ dlogits, const double* scale,
                                                            double* __restrict__ rowloss) {
    __shared__ double sh[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int cnt = 0;
    for (int r = threadIdx.x; r < R; r += blockDim.x) cnt += labels[r] >= 0;
    const double B = block_sum_d(static_cast<double>(cnt), sh);
    if (blockIdx.x == 0 && threadIdx.x == 0) rowloss[R] = B;
    const double gs = scale ? *scale : 1.0;
    const float g = B > 0 ? static_cast<float>(1.0 * gs / B) : 0.f;
    const int r = blockIdx.x * kRowsPerCta + wid;
    if (r >= R) return;
    const int y = labels[r];
    const T* x = logits + static_cast<int64_t>(r) * ld;
    T* dx = dlogits + static_cast<int64_t>(r) * ld;
    if (y < 0) {
        for (int j = lane; j < ld; j += 32) dx[j] = from_f<T>(0.f);
        if (lane == 0) rowloss[r] = 0.0;
        return;
    }
    double mx = -INFINITY;
    for (int j = lane; j < ncls; j += 32) mx = fmax(mx, static_cast<double>(ldv(x, j)));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double z = 0.0;
    for (int j = lane; j < ncls; j += 32) z += exp(static_cast<double>(ldv(x, j)) - mx);
    z = warp_sum(z);
    float py = 0.f;
    for (int j = lane; j < ld; j += 32) {
        if (j < ncls) {
            const float pj = static_cast<float>(exp(static_cast<double>(ldv(x, j)) - mx) / z);
            if (j == y) py = pj;
            dx[j] = from_f<T>((pj - (j == y ? 1.0f : 0.0f)) * g);
        } else {
            dx[j] = from_f<T>(0.f);
        }
    }
    py = __shfl_sync(0xffffffffu, py, y & 31);
    if (lane == 0) rowloss[r] = -log(fmax(1e-30, static_cast<double>(py)));
}

template <class T>
__global__ void __launch_bounds__(256) rcnn_sl1_mc_kernel(const T* __restrict__ pred, int R, int ld,
                                                          const int32_t* __restrict__ labels,
                                                          const float* __restrict__ targets, double beta,
                                                          T* __restrict__ dp, const double* scale,
                                                          double* __restrict__ partial) {
    __shared__ double sh[32];
    int cnt = 0;
    for (int r = threadIdx.x; r < R; r += blockDim.x) cnt += labels[r] >= 0;
    const double norm = block_sum_d(static_cast<double>(cnt), sh);
    if (blockIdx.x == 0 && threadIdx.x == 0) partial[gridDim.x] = norm;
    const double gs = (scale ? *scale : 1.0) / (norm > 0 ? norm : 1.0);
    double acc = 0.0;
    const int r0 = blockIdx.x * kRowsPerCta;
    const int r1 = min(R, r0 + kRowsPerCta);
    for (int64_t i = static_cast<int64_t>(r0) * ld + threadIdx.x; i < static_cast<int64_t>(r1) * ld; i += blockDim.x) {
        const int r = static_cast<int>(i / ld), col = static_cast<int>(i % ld);
        const int lab = labels[r];
        float gout = 0.f;
        if (lab > 0 && col >= 4 * lab && col < 4 * lab + 4) {
            const double d = static_cast<double>(ldv(pred, i)) - static_cast<double>(targets[r * 4 + (col - 4 * lab)]);
            double l, gg;
            sl1(d, beta, l, gg);
            acc += l;
            gout = static_cast<float>(gg * gs);
        }
        dp[i] = from_f<T>(gout);
    }
    const double tot = block_sum_d(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// loss = sum(v[0..n)) / v[n], fixed order: lane-strided partial sums, then an
// in-order sum of the 32 lane totals by lane 0
__global__ void ordered_mean_kernel(const double* __restrict__ v, int n, double* loss_out, int slot) {
    __shared__ double t[32];
    double a = 0.0;
    for (int i = threadIdx.x; i < n; i += 32) a += v[i];
    t[threadIdx.x] = a;
    __syncwarp();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < 32; ++i) s += t[i];
        const double d = v[n];
        loss_out[slot] = d > 0 ? s / d : 0.0;
    }
}

template <class T>
__global__ void __launch_bounds__(kLossBlockThreads) rpn_sl1_kernel(const T* __restrict__ deltas, int64_t n_loc, int A,
                                                                    int A_pad, const int8_t* __restrict__ labels,
                                                                    const float* __restrict__ targets, double beta,
                                                                    double norm, T* __restrict__ dd, const double* scale,
                                                                    double* __restrict__ partial) {
    __shared__ double sh[8];
    const int64_t n = n_loc * 4 * A_pad;
    const double gs = (scale ? *scale : 1.0) / norm;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t loc = i / (4 * A_pad);
        const int rem = static_cast<int>(i % (4 * A_pad));
        const int a = rem / 4, k = rem % 4;
        float gout = 0.f;
        if (a < A && labels[loc * A + a] == 1) {
            const double d = static_cast<double>(ldv(deltas, i)) - static_cast<double>(targets[(loc * A + a) * 4 + k]);
            double l, g;
            sl1(d, beta, l, g);
            acc += l;
            gout = static_cast<float>(g * gs);
        }
        dd[i] = from_f<T>(gout);
    }
    const double tot = block_sum_d256(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

template <class T>
__global__ void __launch_bounds__(kLossThreads) rcnn_sl1_kernel(const T* __restrict__ pred, int R, int ld,
                                                                const int32_t* __restrict__ labels,
                                                                const float* __restrict__ targets, double beta,
                                                                T* __restrict__ dp, const double* scale,
                                                                double* loss_out, int slot) {
    __shared__ double sh[32];
    int cnt = 0;
    for (int r = threadIdx.x; r < R; r += blockDim.x) cnt += labels[r] >= 0;
    const double norm = block_sum_d(static_cast<double>(cnt), sh);
    const double gs = (scale ? *scale : 1.0) / (norm > 0 ? norm : 1.0);
    double acc = 0.0;
    const int64_t n = static_cast<int64_t>(R) * ld;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int r = static_cast<int>(i / ld), col = static_cast<int>(i % ld);
        const int lab = labels[r];
        float gout = 0.f;
        if (lab > 0 && col >= 4 * lab && col < 4 * lab + 4) {
            const double d = static_cast<double>(ldv(pred, i)) - static_cast<double>(targets[r * 4 + (col - 4 * lab)]);
            double l, g;
            sl1(d, beta, l, g);
            acc += l;
            gout = static_cast<float>(g * gs);
        }
        dp[i] = from_f<T>(gout);
    }
    const double tot = block_sum_d(acc, sh);
    if (threadIdx.x == 0) loss_out[slot] = norm > 0 ? tot / norm : 0.0;
}

// ---------------------------------------------------------------- synthetic images
SDB_DEV uint64_t mix64d(uint64_t a, uint64_t b) {
    uint64_t z = a ^ (b + 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// reference image layout [N][3][H][W] -> device NHWC with channels padded to Cp
// (zeros), one pixel per thread, one 16-byte store per pixel for fp16/Cp = 8
template <class T>
__global__ void nchw3_to_nhwc_kernel(const T* __restrict__ in, int n, int H, int W, int Cp, T* __restrict__ out) {
    const int64_t hw = static_cast<int64_t>(H) * W, total = static_cast<int64_t>(n) * hw;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t img = e / hw, px = e - img * hw;
        const T* src = in + img * 3 * hw + px;
        T* o = out + e * Cp;
        o[0] = src[0];
        o[1] = src[hw];
        o[2] = src[2 * hw];
        for (int c = 3; c < Cp; ++c) o[c] = from_f<T>(0.f);
    }
}

template <class T>
__global__ void synth_kernel(T* __restrict__ out, int n, int H, int W, int Cp, uint64_t seed,
                             const int64_t* __restrict__ slots, int64_t slot0) {
    const int64_t total = static_cast<int64_t>(n) * H * W;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int img = static_cast<int>(e / (static_cast<int64_t>(H) * W));
        const int64_t hw = e % (static_cast<int64_t>(H) * W);
        const int64_t slot = slots ? slots[img] : slot0 + img;
        const uint64_t key = mix64d(seed ^ 0x1a2b3c4d5e6f7788ull, static_cast<uint64_t>(slot));
        T* o = out + e * Cp;
        for (int c = 0; c < Cp; ++c) {
            float v = 0.f;
            if (c < 3) {
                const uint64_t el = static_cast<uint64_t>(c) * H * W + hw;
                const uint64_t r1 = mix64d(key, 2 * el), r2 = mix64d(key, 2 * el + 1);
                const float u1 = (static_cast<float>(r1 >> 40) + 0.5f) * 0x1.0p-24f;
                const float u2 = static_cast<float>(r2 >> 40) * 0x1.0p-24f;
                v = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
            }
            o[c] = from_f<T>(v);
        }
    }
}

int grid_for(int64_t n) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 16 * kNumSMs)));
}

}  // namespace

#define SDB_DISPATCH(dtype, KERNEL, GRID, BLOCK, SMEM, ST, ...)                         \
    do {                                                                                \
        if ((dtype) == kF16) KERNEL<__half><<<GRID, BLOCK, SMEM, ST>>>(__VA_ARGS__);    \
        else KERNEL<float><<<GRID, BLOCK, SMEM, ST>>>(__VA_ARGS__);                     \
    } while (0)

template <class T>
static inline const T* cp(const void* p) { return static_cast<const T*>(p); }

// shared memory of the staged forward: the image's feature slab, its RoI list
// and one chunk's sample table
static size_t ra_fwd_smem(int H, int W, int R, int Po, int sr, int dtype) {
    return static_cast<size_t>(H) * W * 8 * (dtype == kF16 ? 2 : 4) + static_cast<size_t>((R + 3) & ~3) * 4 +
           static_cast<size_t>(kRaChunk) * 2 * Po * sr * sizeof(RaTab);
}

template <class T, int SR>
static void ra_fwd_launch(dim3 grid, size_t smem, const void* feat, int H, int W, int C, const float* rois, int R,
                          int P, float scale, int sr, int step, void* out, cudaStream_t st) {
    auto k = roialign_fwd_smem_kernel<T, SR>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k<<<grid, kRaFwdThreads, smem, st>>>(cp<T>(feat), H, W, C, rois, R, P, scale, sr, step, static_cast<T*>(out));
}

cudaError_t roialign_fwd(int dtype, const void* feat, int N, int H, int W, int C, const float* rois, int R, int P,
                         float scale, int sr, void* out, cudaStream_t st, int step) {
    if (step < 1) return cudaErrorInvalidValue;
    if (R == 0) return cudaSuccess;
    const int Po = (P + step - 1) / step;
    if (sr == 2 && C % 8 == 0) {
        const int64_t warps = static_cast<int64_t>(R) * Po * ((C + 255) / 256);
        const unsigned blocks = static_cast<unsigned>((warps + kRaWarps - 1) / kRaWarps);
        if (dtype == kF16)
            roialign_fwd_warp_kernel<__half, 2><<<blocks, 32 * kRaWarps, 0, st>>>(
                cp<__half>(feat), H, W, C, rois, R, P, scale, step, static_cast<__half*>(out));
        else
            roialign_fwd_warp_kernel<float, 2><<<blocks, 32 * kRaWarps, 0, st>>>(
                cp<float>(feat), H, W, C, rois, R, P, scale, step, static_cast<float*>(out));
        return cudaGetLastError();
    }
    // other sampling ratios: the smem-staged slab kernel
    const size_t smem = ra_fwd_smem(H, W, R, Po, sr, dtype);
    if (smem <= 200 * 1024 && sr <= 8) {
        const dim3 grid(C / 8, N);
        const bool h = dtype == kF16;
        if (sr == 2)
            h ? ra_fwd_launch<__half, 2>(grid, smem, feat, H, W, C, rois, R, P, scale, sr, step, out, st)
              : ra_fwd_launch<float, 2>(grid, smem, feat, H, W, C, rois, R, P, scale, sr, step, out, st);
        else
            h ? ra_fwd_launch<__half, 0>(grid, smem, feat, H, W, C, rois, R, P, scale, sr, step, out, st)
              : ra_fwd_launch<float, 0>(grid, smem, feat, H, W, C, rois, R, P, scale, sr, step, out, st);
        return cudaGetLastError();
    }
    // feature maps too large to stage: one thread per (RoI, bin, 8 channels) through L2
    const int64_t total = static_cast<int64_t>(R) * Po * Po * (C / 8);
    if (dtype == kF16)
        roialign_fwd_kernel<__half><<<grid_for(total), 256, 0, st>>>(cp<__half>(feat), H, W, C, rois, R, P, scale, sr,
                                                                    step, static_cast<__half*>(out));
    else
        roialign_fwd_kernel<float><<<grid_for(total), 256, 0, st>>>(cp<float>(feat), H, W, C, rois, R, P, scale, sr,
                                                                   step, static_cast<float*>(out));
    return cudaGetLastError();
}

static int ra_table_width(int P, int step) { return (P + step - 1) / step <= 8 ? 8 : 16; }

// backward workspace: weight table, boxes, nonzero-bin counts, then the block
// plan (lists, segment starts, segment table, partial slots, tickets, partials)
struct RaBwdWs {
    float* tab;
    int4* box;
    uint8_t* nzc;
    int *tl_cnt, *tl_nseg, *seg_start, *tl, *seg, *nseg_total, *slot;
    unsigned* ticket;
    float* part;
    size_t bytes;
};

static RaBwdWs ra_bwd_ws(void* base, int R, int H, int W, int P, int step, int N, int C) {
    auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
    const int pw = ra_table_width(P, step);
    const size_t nt = static_cast<size_t>((H + kRaBlk - 1) / kRaBlk) * ((W + kRaBlk - 1) / kRaBlk) * std::max(N, 1);
    const int V = C >= 2048 ? 4 : (C >= 512 ? 2 : 1);
    const size_t nch = static_cast<size_t>((std::max(C, 1) + 256 * V - 1) / (256 * V));
    RaBwdWs w{};
    uint8_t* p = static_cast<uint8_t*>(base);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        uint8_t* q = p ? p + off : nullptr;
        off += al(bytes);
        return q;
    };
    w.tab = reinterpret_cast<float*>(take(static_cast<size_t>(R) * (H + W) * pw * 4));
    w.box = reinterpret_cast<int4*>(take(static_cast<size_t>(R) * 16));
    w.nzc = take(static_cast<size_t>(R) * (H + W));
    w.tl_cnt = reinterpret_cast<int*>(take(nt * 4));
    w.tl_nseg = reinterpret_cast<int*>(take(nt * 4));
    w.seg_start = reinterpret_cast<int*>(take(nt * (kRaSegMax + 1) * 4));
    w.seg = reinterpret_cast<int*>(take(nt * kRaSegMax * 4));
    w.nseg_total = reinterpret_cast<int*>(take(4));
    w.slot = reinterpret_cast<int*>(take(nt * 4));
    w.ticket = reinterpret_cast<unsigned*>(take(nt * nch * 4));
    w.part = reinterpret_cast<float*>(take(static_cast<size_t>(kRaSlots) * nch * kRaBlk * kRaBlk * 256 * V * 4));
    w.tl = reinterpret_cast<int*>(take(nt * static_cast<size_t>(std::max(R, 1)) * 4));
    w.bytes = off + 256;
    return w;
}

// C is not a parameter of the reference-shaped query: size for C <= 2048 (V = 4)
size_t roialign_bwd_workspace(int R, int H, int W, int P, int step, int N) {
    if (step < 1) return 0;
    return ra_bwd_ws(nullptr, R, H, W, P, step, N, 2048).bytes;
}

cudaError_t roialign_bwd(int dtype, const void* dy, int N, int H, int W, int C, const float* rois, int R, int P,
                         float scale, int sr, void* dfeat, void* ws, size_t ws_bytes, cudaStream_t st, int step) {
    if (step < 1 || (P + step - 1) / step > 16) return cudaErrorInvalidValue;
    if (ws_bytes < roialign_bwd_workspace(R, H, W, P, step, N)) return cudaErrorInvalidValue;
    const int Po = (P + step - 1) / step, pw = ra_table_width(P, step);
    const RaBwdWs w = ra_bwd_ws(ws, R, H, W, P, step, N, C);
    if (R > 0)
        roialign_bwd_weights_kernel<<<(R + 7) / 8, 256, 0, st>>>(rois, R, H, W, P, scale, sr, step, pw, w.tab, w.box,
                                                                 w.nzc);
    const int ntiles = ((H + kRaBlk - 1) / kRaBlk) * ((W + kRaBlk - 1) / kRaBlk), nt = N * ntiles;
    const size_t lsm = static_cast<size_t>(std::max(R, 1)) * 4;
    static int lsm_set = 0;
    if (lsm > 48 * 1024 && lsm > static_cast<size_t>(lsm_set)) {
        cudaFuncSetAttribute(roialign_tile_list_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(lsm));
        lsm_set = static_cast<int>(lsm);
    }
    // segment work target: kRaSegWork pairs at 7 x 7 pooled bins, scaled with the bin count
    const long long seg_work = std::max<long long>(kRaSegWork, static_cast<long long>(kRaSegWork) * Po * Po / 49);
    roialign_tile_list_kernel<<<dim3(ntiles, N), 256, lsm, st>>>(w.box, w.nzc, R, H, W, seg_work, w.tl_cnt,
                                                                  w.tl_nseg, w.seg_start, w.tl);
    // channel slab per warp: 256*V channels (V 8-channel chunks per lane)
    const int V = C >= 2048 ? 4 : (C >= 512 ? 2 : 1);
    const int nch = (C + 256 * V - 1) / (256 * V);
    roialign_seg_plan_kernel<<<1, 1024, 0, st>>>(w.tl_nseg, nt, w.seg, w.nseg_total, w.slot, w.ticket, nt * nch);
    const dim3 grid(static_cast<unsigned>(std::min(nt * 2, 4 * kNumSMs)), nch);
    const float inv = 1.0f / static_cast<float>(max(sr * sr, 1));
    const bool h = dtype == kF16;
    auto go = [&](auto kern, auto* dyp, auto* dxp) {
        kern<<<grid, kRaBlk * kRaBlk * 32, 0, st>>>(dyp, H, W, C, w.box, w.tab, R, Po, pw, inv, dxp, w.tl_cnt,
                                                   w.tl_nseg, w.seg_start, w.tl, w.seg, w.nseg_total, w.slot, w.ticket,
                                                   w.part);
    };
    if (V == 4) h ? go(roialign_bwd_gather_kernel<__half, 4>, cp<__half>(dy), static_cast<__half*>(dfeat))
                  : go(roialign_bwd_gather_kernel<float, 4>, cp<float>(dy), static_cast<float*>(dfeat));
    else if (V == 2) h ? go(roialign_bwd_gather_kernel<__half, 2>, cp<__half>(dy), static_cast<__half*>(dfeat))
                       : go(roialign_bwd_gather_kernel<float, 2>, cp<float>(dy), static_cast<float*>(dfeat));
    else h ? go(roialign_bwd_gather_kernel<__half, 1>, cp<__half>(dy), static_cast<__half*>(dfeat))
           : go(roialign_bwd_gather_kernel<float, 1>, cp<float>(dy), static_cast<float*>(dfeat));
    return cudaGetLastError();
}

// 32-bit element indexing when the grid-stride range fits (with room for the stride step)
template <class F>
void launch_idx(int64_t total, F&& f) {
    if (total + static_cast<int64_t>(grid_for(total)) * 256 < (int64_t{1} << 31)) f(int32_t{0});
    else f(int64_t{0});
}

cudaError_t maxpool_fwd(int dtype, const void* x, int N, int H, int W, int C, int k, int s, int p, void* y,
                        uint8_t* argmax, cudaStream_t st) {
    const int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
    const int64_t total = static_cast<int64_t>(N) * Ho * Wo * (C / 8);
    static const bool generic = std::getenv("SDB_MAXPOOL_GENERIC") != nullptr;  // A/B switch
    if (k == 3 && s == 2 && p == 1 && static_cast<int64_t>(N) * Ho < 65536 && !generic) {
        const dim3 grid((Wo * (C / 8) + 255) / 256, N * Ho);
        if (dtype == kF16)
            maxpool_fwd_k3s2_kernel<__half><<<grid, 256, 0, st>>>(cp<__half>(x), H, W, C / 8, Ho, Wo,
                                                                  static_cast<__half*>(y), argmax);
        else
            maxpool_fwd_k3s2_kernel<float><<<grid, 256, 0, st>>>(cp<float>(x), H, W, C / 8, Ho, Wo,
                                                                 static_cast<float*>(y), argmax);
        return cudaGetLastError();
    }
    if (dtype == kF16)
        launch_idx(total, [&](auto idx) {
            maxpool_fwd_kernel<__half, decltype(idx)><<<grid_for(total), 256, 0, st>>>(
                cp<__half>(x), N, H, W, C, k, s, p, Ho, Wo, static_cast<__half*>(y), argmax);
        });
    else
        launch_idx(total, [&](auto idx) {
            maxpool_fwd_kernel<float, decltype(idx)><<<grid_for(total), 256, 0, st>>>(
                cp<float>(x), N, H, W, C, k, s, p, Ho, Wo, static_cast<float*>(y), argmax);
        });
    return cudaGetLastError();
}

cudaError_t maxpool_bwd(int dtype, const void* dy, const uint8_t* argmax, int N, int H, int W, int C, int k, int s,
                        int p, void* dx, cudaStream_t st) {
    const int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
    const int64_t total = static_cast<int64_t>(N) * H * W * (C / 8);
    static const bool generic = std::getenv("SDB_MAXPOOL_GENERIC") != nullptr;  // A/B switch
    if (k == 3 && s == 2 && p == 1 && static_cast<int64_t>(N) * H < 65536 && !generic) {
        const dim3 grid((W * (C / 8) + 255) / 256, N * H);
        if (dtype == kF16)
            maxpool_bwd_k3s2_kernel<__half><<<grid, 256, 0, st>>>(cp<__half>(dy), argmax, H, W, C / 8, Ho, Wo,
                                                                  static_cast<__half*>(dx));
        else
            maxpool_bwd_k3s2_kernel<float><<<grid, 256, 0, st>>>(cp<float>(dy), argmax, H, W, C / 8, Ho, Wo,
                                                                 static_cast<float*>(dx));
        return cudaGetLastError();
    }
    if (dtype == kF16)
        launch_idx(total, [&](auto idx) {
            maxpool_bwd_kernel<__half, decltype(idx)><<<grid_for(total), 256, 0, st>>>(
                cp<__half>(dy), argmax, N, H, W, C, k, s, p, Ho, Wo, static_cast<__half*>(dx));
        });
    else
        launch_idx(total, [&](auto idx) {
            maxpool_bwd_kernel<float, decltype(idx)><<<grid_for(total), 256, 0, st>>>(
                cp<float>(dy), argmax, N, H, W, C, k, s, p, Ho, Wo, static_cast<float*>(dx));
        });
    return cudaGetLastError();
}

cudaError_t avgpool_fwd(int dtype, const void* x, int N, int HW, int C, void* y, cudaStream_t st) {
    const int64_t total = static_cast<int64_t>(N) * (C / 8);
    if (dtype == kF16)
        avgpool_fwd_kernel<__half><<<grid_for(total), 256, 0, st>>>(cp<__half>(x), N, HW, C, static_cast<__half*>(y));
    else
        avgpool_fwd_kernel<float><<<grid_for(total), 256, 0, st>>>(cp<float>(x), N, HW, C, static_cast<float*>(y));
    return cudaGetLastError();
}

cudaError_t avgpool_bwd(int dtype, const void* dy, int N, int HW, int C, void* dx, cudaStream_t st, const void* act_y,
                        float neg, const uint8_t* act_bits) {
    const int64_t total = static_cast<int64_t>(N) * HW * (C / 8);
    const float inv = static_cast<float>(1.0 / static_cast<double>(HW));  // src/autograd.cpp:381-384
    if (dtype == kF16)
        launch_idx(total, [&](auto idx) {
            avgpool_bwd_kernel<__half, decltype(idx)><<<grid_for(total), 256, 0, st>>>(
                cp<__half>(dy), N, HW, C, inv, static_cast<__half*>(dx), cp<__half>(act_y), neg, act_bits);
        });
    else
        launch_idx(total, [&](auto idx) {
            avgpool_bwd_kernel<float, decltype(idx)><<<grid_for(total), 256, 0, st>>>(
                cp<float>(dy), N, HW, C, inv, static_cast<float*>(dx), cp<float>(act_y), neg, act_bits);
        });
    return cudaGetLastError();
}

cudaError_t add_act(int dtype, const void* a, const void* b, void* out, int64_t n, int act, float slope,
                    cudaStream_t st) {
    const int64_t n8 = n / 8;
    if (dtype == kF16)
        add_act_kernel<__half><<<grid_for(n8), 256, 0, st>>>(cp<__half>(a), cp<__half>(b), static_cast<__half*>(out),
                                                             n8, act, slope);
    else
        add_act_kernel<float><<<grid_for(n8), 256, 0, st>>>(cp<float>(a), cp<float>(b), static_cast<float*>(out), n8,
                                                            act, slope);
    return cudaGetLastError();
}

cudaError_t act_bwd(int dtype, const void* dy, const void* y, void* dx, int64_t n, float neg, cudaStream_t st) {
    const int64_t n8 = n / 8;
    if (dtype == kF16)
        act_bwd_kernel<__half><<<grid_for(n8), 256, 0, st>>>(cp<__half>(dy), cp<__half>(y), static_cast<__half*>(dx),
                                                             n8, neg);
    else
        act_bwd_kernel<float><<<grid_for(n8), 256, 0, st>>>(cp<float>(dy), cp<float>(y), static_cast<float*>(dx), n8,
                                                            neg);
    return cudaGetLastError();
}

cudaError_t relu_fwd(int dtype, const void* x, void* y, int64_t n, cudaStream_t st) {
    const int64_t n8 = n / 8;
    if (dtype == kF16) relu_kernel<__half><<<grid_for(n8), 256, 0, st>>>(cp<__half>(x), static_cast<__half*>(y), n8);
    else relu_kernel<float><<<grid_for(n8), 256, 0, st>>>(cp<float>(x), static_cast<float*>(y), n8);
    return cudaGetLastError();
}

cudaError_t add_inplace(int dtype, void* acc, const void* b, int64_t n, cudaStream_t st) {
    const int64_t n8 = n / 8;
    if (dtype == kF16)
        add_inplace_kernel<__half><<<grid_for(n8), 256, 0, st>>>(static_cast<__half*>(acc), cp<__half>(b), n8);
    else
        add_inplace_kernel<float><<<grid_for(n8), 256, 0, st>>>(static_cast<float*>(acc), cp<float>(b), n8);
    return cudaGetLastError();
}

size_t loss_workspace_bytes(int64_t) { return 3 * kLossBlocks * sizeof(double); }

cudaError_t softmax_ce(int dtype, const void* logits, int R, int ncls, int ld, const int32_t* labels, void* dlogits,
                       const LossArgs& la, void* ws, cudaStream_t st) {
    if (ws && R > 0) {
        // ws: R + 1 doubles (per-row losses, then the valid-row count)
        double* rl = static_cast<double*>(ws);
        const int g = (R + kRowsPerCta - 1) / kRowsPerCta;
        if (dtype == kF16)
            softmax_ce_mc_kernel<__half><<<g, 256, 0, st>>>(cp<__half>(logits), R, ncls, ld, labels,
                                                            static_cast<__half*>(dlogits), la.scale, rl);
        else
            softmax_ce_mc_kernel<float><<<g, 256, 0, st>>>(cp<float>(logits), R, ncls, ld, labels,
                                                           static_cast<float*>(dlogits), la.scale, rl);
        ordered_mean_kernel<<<1, 32, 0, st>>>(rl, R, la.loss_out, la.slot);
        return cudaGetLastError();
    }
    if (dtype == kF16)
        softmax_ce_kernel<__half><<<1, kLossThreads, 0, st>>>(cp<__half>(logits), R, ncls, ld, labels,
                                                             static_cast<__half*>(dlogits), la.scale, la.loss_out,
                                                             la.slot);
    else
        softmax_ce_kernel<float><<<1, kLossThreads, 0, st>>>(cp<float>(logits), R, ncls, ld, labels,
                                                            static_cast<float*>(dlogits), la.scale, la.loss_out, la.slot);
    return cudaGetLastError();
}

cudaError_t sigmoid_bce(int dtype, const void* logits, int64_t n_loc, int A, int A_pad, const int8_t* labels,
                        void* dlogits, const LossArgs& la, void* ws, cudaStream_t st) {
    double* counts = static_cast<double*>(ws);
    double* partial = counts + kLossBlocks;
    label_count_kernel<<<kLossBlocks, kLossBlockThreads, 0, st>>>(labels, n_loc * A, counts);
    if (dtype == kF16)
        sigmoid_bce_kernel<__half><<<kLossBlocks, kLossBlockThreads, 0, st>>>(
            cp<__half>(logits), n_loc, A, A_pad, labels, static_cast<__half*>(dlogits), la.scale, counts, partial);
    else
        sigmoid_bce_kernel<float><<<kLossBlocks, kLossBlockThreads, 0, st>>>(
            cp<float>(logits), n_loc, A, A_pad, labels, static_cast<float*>(dlogits), la.scale, counts, partial);
    loss_finalize_kernel<<<1, 32, 0, st>>>(partial, kLossBlocks, counts, 0.0, la.loss_out, la.slot);
    return cudaGetLastError();
}

cudaError_t rpn_smooth_l1(int dtype, const void* deltas, int64_t n_loc, int A, int A_pad, const int8_t* labels,
                          const float* targets, double beta, double norm, void* dd, const LossArgs& la, void* ws,
                          cudaStream_t st) {
    double* partial = static_cast<double*>(ws) + 2 * kLossBlocks;
    if (dtype == kF16)
        rpn_sl1_kernel<__half><<<kLossBlocks, kLossBlockThreads, 0, st>>>(cp<__half>(deltas), n_loc, A, A_pad, labels,
                                                                         targets, beta, norm, static_cast<__half*>(dd),
                                                                         la.scale, partial);
    else
        rpn_sl1_kernel<float><<<kLossBlocks, kLossBlockThreads, 0, st>>>(cp<float>(deltas), n_loc, A, A_pad, labels,
                                                                        targets, beta, norm, static_cast<float*>(dd),
                                                                        la.scale, partial);
    loss_finalize_kernel<<<1, 32, 0, st>>>(partial, kLossBlocks, nullptr, norm, la.loss_out, la.slot);
    return cudaGetLastError();
}

cudaError_t rcnn_smooth_l1(int dtype, const void* pred, int R, int ld, const int32_t* labels, const float* targets,
                           double beta, void* dp, const LossArgs& la, void* ws, cudaStream_t st) {
    if (ws && R > 0) {
        // ws: one fp64 partial per CTA, then the valid-row count
        double* part = static_cast<double*>(ws);
        const int g = (R + kRowsPerCta - 1) / kRowsPerCta;
        if (dtype == kF16)
            rcnn_sl1_mc_kernel<__half><<<g, 256, 0, st>>>(cp<__half>(pred), R, ld, labels, targets, beta,
                                                          static_cast<__half*>(dp), la.scale, part);
        else
            rcnn_sl1_mc_kernel<float><<<g, 256, 0, st>>>(cp<float>(pred), R, ld, labels, targets, beta,
                                                         static_cast<float*>(dp), la.scale, part);
        ordered_mean_kernel<<<1, 32, 0, st>>>(part, g, la.loss_out, la.slot);
        return cudaGetLastError();
    }
    if (dtype == kF16)
        rcnn_sl1_kernel<__half><<<1, kLossThreads, 0, st>>>(cp<__half>(pred), R, ld, labels, targets, beta,
                                                           static_cast<__half*>(dp), la.scale, la.loss_out, la.slot);
    else
        rcnn_sl1_kernel<float><<<1, kLossThreads, 0, st>>>(cp<float>(pred), R, ld, labels, targets, beta,
                                                          static_cast<float*>(dp), la.scale, la.loss_out, la.slot);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- stem as a GEMM
// The 7x7 stride-2 stem sees 3 real input channels (of 8 stored): its im2col
// matrix X' [pixels][192] (column j = r*24 + s*3 + c for c < 3, zeros
// elsewhere) turns fprop and wgrad into 1x1 tensor-core GEMMs with 64-wide
// K blocks (src/tensor.cpp:178-194 semantics; accumulation order differs).
constexpr int kStemK = 7, kStemCols = 192;

// One CTA per (image row of output, 64 output columns): the 7 input rows x
// 133 input columns it needs (3 real channels, read as 8-byte pixel heads) are
// staged in shared memory once, the segment's 64 x 192 output block (one
// contiguous 24 KB run of X') is assembled in shared memory and leaves with a
// single bulk copy.
constexpr int kStemSeg = 64;
__global__ void __launch_bounds__(256) stem_im2col_kernel(const __half* __restrict__ x, int N, int H, int W, int Cs,
                                                          int Ho, int Wo, int stride, int pad,
                                                          __half* __restrict__ out) {
    constexpr int kCols = (kStemSeg - 1) * 2 + kStemK;  // input columns of a segment (stride 2)
    __shared__ uint2 patch[kStemK][kCols];
    __shared__ __align__(128) uint4 ob[kStemSeg * kStemCols / 8];
    const int oh = blockIdx.y % Ho, n = blockIdx.y / Ho;
    const int ow0 = blockIdx.x * kStemSeg;
    const int ih0 = oh * stride - pad, iw0 = ow0 * stride - pad;
    for (int i = threadIdx.x; i < kStemK * kCols; i += blockDim.x) {
        const int rr = i / kCols, cc = i - rr * kCols;
        const int ih = ih0 + rr, iw = iw0 + cc;
        uint2 v = make_uint2(0u, 0u);
        if (ih >= 0 && ih < H && iw >= 0 && iw < W)
            v = *reinterpret_cast<const uint2*>(x + ((static_cast<int64_t>(n) * H + ih) * W + iw) * Cs);
        patch[rr][cc] = v;
    }
    __syncthreads();
    const int npx = min(kStemSeg, Wo - ow0);
    for (int i = threadIdx.x; i < kStemSeg * 8; i += blockDim.x) {
        const int j = i >> 3, r = i & 7;  // output column in the segment, tap row (7 = zero pad chunk)
        __half v[24];
#pragma unroll
        for (int k = 0; k < 24; ++k) v[k] = __float2half_rn(0.f);
        if (r < kStemK) {
#pragma unroll
            for (int q = 0; q < kStemK; ++q) {
                const uint2 u = patch[r][j * stride + q];
                const __half* h = reinterpret_cast<const __half*>(&u);
                v[q * 3] = h[0];
                v[q * 3 + 1] = h[1];
                v[q * 3 + 2] = h[2];
            }
        }
        const uint4* src = reinterpret_cast<const uint4*>(v);
        uint4* o = ob + (j * kStemCols + r * 24) / 8;
        o[0] = src[0];
        o[1] = src[1];
        o[2] = src[2];
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0 && npx > 0) {
        const int64_t px0 = (static_cast<int64_t>(n) * Ho + oh) * Wo + ow0;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + px0 * kStemCols),
                     "r"(smem_u32(ob)), "r"(npx * kStemCols * 2)
                     : "memory");
        bulk_commit();
        bulk_wait_all();
    }
}

// W [K][7][7][Cs] -> W' [K][192] (and the transposed fold of dW' back)
__global__ void stem_wrepack_kernel(const __half* __restrict__ w, int K, int Cs, __half* __restrict__ w2, int fold) {
    const int total = K * kStemK * kStemK * Cs;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int c = e % Cs, rs = (e / Cs) % (kStemK * kStemK), k = e / (Cs * kStemK * kStemK);
        const int r = rs / kStemK, q = rs % kStemK;
        const int j = k * kStemCols + r * 24 + q * 3 + c;
        if (fold) w2[e] = c < 3 ? w[j] : __float2half_rn(0.f);  // here w = dW', w2 = dW (KRSC)
        else if (c < 3) w2[j] = w[e];
    }
}

cudaError_t stem_im2col(const void* x, int N, int H, int W, int Cs, int Ho, int Wo, int stride, int pad, void* out,
                        cudaStream_t st) {
    if (stride != 2) return cudaErrorNotSupported;  // the segment staging assumes the stem's stride
    const dim3 grid((Wo + kStemSeg - 1) / kStemSeg, N * Ho);
    stem_im2col_kernel<<<grid, 256, 0, st>>>(cp<__half>(x), N, H, W, Cs, Ho, Wo, stride, pad,
                                             static_cast<__half*>(out));
    return cudaGetLastError();
}

cudaError_t stem_weights(const void* w, int K, int Cs, void* w2, int fold, cudaStream_t st) {
    if (!fold) {
        const cudaError_t e = cudaMemsetAsync(w2, 0, static_cast<size_t>(K) * kStemCols * 2, st);
        if (e != cudaSuccess) return e;
    }
    const int total = K * kStemK * kStemK * Cs;
    stem_wrepack_kernel<<<(total + 255) / 256, 256, 0, st>>>(cp<__half>(w), K, Cs, static_cast<__half*>(w2), fold);
    return cudaGetLastError();
}

cudaError_t nchw3_to_nhwc(int dtype, const void* in, int n, int H, int W, int Cp, void* out, cudaStream_t st) {
    const int64_t total = static_cast<int64_t>(n) * H * W;
    if (dtype == kF16)
        nchw3_to_nhwc_kernel<__half><<<grid_for(total), 256, 0, st>>>(cp<__half>(in), n, H, W, Cp, static_cast<__half*>(out));
    else
        nchw3_to_nhwc_kernel<float><<<grid_for(total), 256, 0, st>>>(cp<float>(in), n, H, W, Cp, static_cast<float*>(out));
    return cudaGetLastError();
}

cudaError_t synth_images(int dtype, void* out, int n, int H, int W, int Cp, uint64_t seed, const int64_t* slots,
                         int64_t slot0, cudaStream_t st) {
    const int64_t total = static_cast<int64_t>(n) * H * W;
    if (dtype == kF16)
        synth_kernel<__half><<<grid_for(total), 256, 0, st>>>(static_cast<__half*>(out), n, H, W, Cp, seed, slots, slot0);
    else
        synth_kernel<float><<<grid_for(total), 256, 0, st>>>(static_cast<float*>(out), n, H, W, Cp, seed, slots, slot0);
    return cudaGetLastError();
}

}  // namespace sdb
