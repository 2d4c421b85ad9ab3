"""Host mirror of the reference operator API (namespace ``simdet``) on top of
the libsdb C ABI.  Same names, argument meaning and error behaviour as the
reference's C++ functions, so parity tests read like the reference's own
tests; tensors are torch CUDA tensors in the reference layout (NCHW / OIHW),
converted to the library's NHWC / KRSC layout at this boundary (the "parity
shim" of SURVEY.md §8(b)).  torch is plumbing only (allocation, streams);
every arithmetic op runs in libsdb's sm_100a kernels.

Reference entry points mirrored (file:line under /root/reference/proj):
  conv2d                      src/tensor.cpp:169-196
  conv2d_backward             src/autograd.cpp:290-320  (Tape conv2d rule)
  syncbn_forward / _backward  src/syncbn.cpp:21-117     (group == nullptr)
  iabn_forward / _backward    src/memopt.cpp:226-327
  apply_sgd / has_nonfinite   src/trainer.cpp:78-94
  update_scale                src/precision.cpp:45-56
  allreduce_sum               src/comm.cpp:288-315      (CommGroup, NCCL)
and the detection operators the reference lacks (restated semantics,
oracle/restate.cpp): anchors, proposal layer, anchor / proposal targets,
RoIAlign, softmax-CE, sigmoid BCE, smooth-L1.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import F16, F32, check, lib

_P, _I, _L, _F, _D = C.c_void_p, C.c_int, C.c_int64, C.c_float, C.c_double

_SIGS = {
    "sdb_ctx_create": [_I, _I, _I, _P, C.POINTER(_P)],
    "sdb_ctx_destroy": [_P],
    "sdb_synchronize": [_P],
    "sdb_get_nccl_unique_id": [_P],
    "sdb_conv_fprop": [_P, _I, _P, _P, _P] + [_I] * 9 + [_P],
    "sdb_conv_dgrad": [_P, _I, _P, _P, _P] + [_I] * 10 + [_P],
    "sdb_conv_dgrad_act": [_P, _I, _P, _P, _P] + [_I] * 9 + [_P, _P, C.c_float, _P, _P],
    "sdb_syncbn_fwd": [_P, _I] + [_P] * 7 + [_L, _I, _F, _I, _P],
    "sdb_syncbn_bwd": [_P, _I] + [_P] * 11 + [_L, _I, _P],
    "sdb_conv_wgrad": [_P, _I, _P, _P, _P] + [_I] * 9 + [_P],
    "sdb_bn_fwd": [_P, _I, _P, _P, _P, _P, _P, _P, _L, _I, _F, _I, _P],
    "sdb_bn_bwd": [_P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _L, _I, _P],
    "sdb_iabn_fwd": [_P, _I, _P, _P, _P, _P, _P, _P, _L, _I, _F, _F, _P],
    "sdb_iabn_bwd": [_P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _L, _I, _F, _P],
    "sdb_nonfinite": [_P, _I, _P, _L, _P, _P],
    "sdb_fused_sgd": [_P, _I, _P, _P, _P, _P, _L, _F, _F, _P, _D, _P, _P],
    "sdb_update_scale": [_P, _P, _P, _P, _I, _L, _D, _D, _D, _D, _P],
    "sdb_cast": [_P, _I, _P, _I, _P, _L, _P],
    "sdb_make_anchors": [_P, _I, _I, _F, _P, _I, _P, _I, _P, _P],
    "sdb_rpn_proposal": [_P, _I, _P, _P, _P, _I, _I, _I, _I, _I, _D, _I, _F, _F, _P, _P, _P, _P, _P],
    "sdb_roialign_fwd": [_P, _I, _P, _I, _I, _I, _I, _P, _I, _I, _F, _I, _P, _P],
    "sdb_roialign_bwd": [_P, _I, _P, _I, _I, _I, _I, _P, _I, _I, _F, _I, _P, _P],
    "sdb_softmax_ce": [_P, _I, _P, _I, _I, _I, _P, _P, _P, _P, _P],
    "sdb_debug_set": [_I, _I],
    "sdb_rpn_bce": [_P, _I, _P, _L, _I, _I, _P, _P, _P, _P, _P],
    "sdb_rpn_smoothl1": [_P, _I, _P, _L, _I, _I, _P, _P, _D, _D, _P, _P, _P, _P],
    "sdb_smoothl1": [_P, _I, _P, _I, _I, _P, _P, _D, _P, _P, _P, _P],
    "sdb_anchor_targets": [_P, _P, _I, _I, _P, _I, _P, _F, _F, _P, _D, _D, _I, _D, _P, _P, _P],
    "sdb_proposal_targets": [_P, _P, _I, _P, _P, _P, _I, _P, _I, _P, _D, _D, _D, _I, _D, _P, _P, _P, _P, _P],
    "sdb_allreduce_sum": [_P, _I, _P, _L, _P],
    "sdb_comm_check": [_P],
    "sdb_conv_fprop_stats": [_P, _I, _P, _P, _P] + [_I] * 9 + [_F, _I, _P, _P, _P, _P],
    "sdb_conv_dgrad_iabn_bwd": [_P, _I, _P, _P, _P] + [_I] * 8 + [_P, _P, _P, _P, _F, _P, _P, _P, _P, _P],
    "sdb_roialign_fwd_folded": [_P, _I, _P, _I, _I, _I, _I, _P, _I, _I, _F, _I, _I, _P, _P],
    "sdb_roialign_bwd_folded": [_P, _I, _P, _I, _I, _I, _I, _P, _I, _I, _F, _I, _I, _P, _P],
}

_configured = False
_ctx = {}


def L():
    global _configured
    lb = lib()
    if not _configured:
        for name, args in _SIGS.items():
            fn = getattr(lb, name)
            fn.argtypes = args
            fn.restype = C.c_int
        _configured = True
    return lb


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise RuntimeError("libsdb ops need CUDA tensors (no CPU fallback)")


def ctx(device: int | None = None):
    """Per-device default context (single rank)."""
    if device is None:
        device = torch.cuda.current_device()
    if device not in _ctx:
        h = _P()
        check(L().sdb_ctx_create(device, 0, 1, None, C.byref(h)))
        _ctx[device] = h
    return _ctx[device]


def stream():
    """torch's current stream; the legacy default stream (handle 0) is passed
    as cudaStreamLegacy (0x1) because a NULL stream means "the context's own
    stream" at the C ABI."""
    h = torch.cuda.current_stream().cuda_stream
    return _P(h if h else 1)


def ptr(t):
    return None if t is None else _P(t.data_ptr())


def dt(t) -> int:
    if t.dtype == torch.float16:
        return F16
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def nchw_to_nhwc(t):
    return t.permute(0, 2, 3, 1).contiguous()


def nhwc_to_nchw(t):
    return t.permute(0, 3, 1, 2).contiguous()


# ------------------------------------------------------------------ NHWC primitives
def conv_fprop_nhwc(x, w, stride, pad):
    _require_cuda(x, w)
    N, H, W, Cc = x.shape
    K, R, S, C2 = w.shape
    Ho = (H + 2 * pad - R) // stride + 1 if H + 2 * pad >= R else 0
    Wo = (W + 2 * pad - S) // stride + 1 if W + 2 * pad >= S else 0
    y = torch.empty((N, max(Ho, 1), max(Wo, 1), K), device=x.device, dtype=x.dtype)
    check(L().sdb_conv_fprop(ctx(), dt(x), ptr(x), ptr(w), ptr(y), N, H, W, Cc, K, R, S, stride, pad, stream()))
    return y


def conv_fprop_stats_nhwc(x, w, stride, pad, eps=1e-5, iabn=False):
    """fprop + the following norm layer's statistics (fused into the epilogue on
    the TMA-store path); returns (y, mean, invstd, fused)"""
    _require_cuda(x, w)
    N, H, W, Cc = x.shape
    K, R, S, _ = w.shape
    Ho, Wo = (H + 2 * pad - R) // stride + 1, (W + 2 * pad - S) // stride + 1
    y = torch.empty((N, Ho, Wo, K), device=x.device, dtype=x.dtype)
    mean = torch.empty(K, device=x.device, dtype=torch.float32)
    invstd = torch.empty_like(mean)
    fused = C.c_int(0)
    check(L().sdb_conv_fprop_stats(ctx(), dt(x), ptr(x), ptr(w), ptr(y), N, H, W, Cc, K, R, S, stride, pad, eps,
                                   1 if iabn else 0, ptr(mean), ptr(invstd), C.byref(fused), stream()))
    return y, mean, invstd, bool(fused.value)


def conv_dgrad_iabn_bwd_nhwc(dy, w, y, gamma, beta, invstd, slope, pad):
    """stride-1 dgrad producing the gradient of the IABN output y, then that
    layer's IABN backward (statistics fused into the dgrad epilogue on the
    tensor-core path); returns (dy_iabn, dz, dgamma, dbeta, fused)"""
    _require_cuda(dy, w, y)
    N, H, W, Cc = y.shape
    K, R, S, _ = w.shape
    dyi = torch.empty_like(y)
    dz = torch.empty_like(y)
    dgamma = torch.empty(Cc, device=y.device, dtype=torch.float32)
    dbeta = torch.empty_like(dgamma)
    fused = C.c_int(0)
    check(L().sdb_conv_dgrad_iabn_bwd(ctx(), dt(y), ptr(dy), ptr(w), ptr(dyi), N, H, W, Cc, K, R, S, pad, ptr(y),
                                      ptr(gamma), ptr(beta), ptr(invstd), slope, ptr(dz), ptr(dgamma), ptr(dbeta),
                                      C.byref(fused), stream()))
    return dyi, dz, dgamma, dbeta, bool(fused.value)


def conv_dgrad_nhwc(dy, w, x_shape, stride, pad, out=None, accumulate=False):
    N, H, W, Cc = x_shape
    K, R, S, _ = w.shape
    dx = out if out is not None else torch.empty((N, H, W, Cc), device=dy.device, dtype=dy.dtype)
    check(L().sdb_conv_dgrad(ctx(), dt(dy), ptr(dy), ptr(w), ptr(dx), N, H, W, Cc, K, R, S, stride, pad,
                             1 if accumulate else 0, stream()))
    return dx


def sign_bits_nhwc(y):
    """sign bitmap of an NHWC tensor: bit c%8 of byte [pixel][c/8] = (y > 0)"""
    b = (y.reshape(-1, y.shape[-1] // 8, 8) > 0).to(torch.int32)
    w8 = torch.tensor([1 << j for j in range(8)], dtype=torch.int32, device=y.device)
    return (b * w8).sum(-1).to(torch.uint8).contiguous()


def conv_dgrad_act_nhwc(dy, w, addend, y, neg, stride, pad, y_bits=None):
    """dx = act'(y) * rn16(conv^T(dy, w) + addend): the step's fused residual + activation backward"""
    N, H, W, Cc = y.shape
    K, R, S, _ = w.shape
    dx = torch.empty((N, H, W, Cc), device=dy.device, dtype=dy.dtype)
    check(L().sdb_conv_dgrad_act(ctx(), dt(dy), ptr(dy), ptr(w), ptr(dx), N, H, W, Cc, K, R, S, stride, pad,
                                 ptr(addend), ptr(y), float(neg), ptr(y_bits) if y_bits is not None else None,
                                 stream()))
    return dx


def conv_wgrad_nhwc(x, dy, w_shape, stride, pad):
    N, H, W, Cc = x.shape
    K, R, S, _ = w_shape
    dw = torch.empty((K, R, S, Cc), device=x.device, dtype=x.dtype)
    check(L().sdb_conv_wgrad(ctx(), dt(x), ptr(x), ptr(dy), ptr(dw), N, H, W, Cc, K, R, S, stride, pad, stream()))
    return dw


# ------------------------------------------------------------------ reference-shaped API
def conv2d(x, k, stride: int, pad: int):
    """simdet::conv2d (src/tensor.cpp:169): x [N,C,H,W], k [O,C,kh,kw]."""
    from . import ShapeError
    if x.dim() != 4 or k.dim() != 4:
        raise ShapeError("conv2d: rank-4 operands required")
    if x.dtype != k.dtype:
        raise ShapeError("conv2d: dtype mismatch")
    if x.shape[1] != k.shape[1]:
        raise ShapeError("conv2d: channel mismatch")
    y = conv_fprop_nhwc(nchw_to_nhwc(x), nchw_to_nhwc(k), stride, pad)
    return nhwc_to_nchw(y)


def conv2d_backward(x, k, dy, stride: int, pad: int):
    """Tape conv2d backward rule (src/autograd.cpp:290-320) + leaf-dtype finalisation."""
    dy = dy.to(x.dtype)
    xn, kn, dyn = nchw_to_nhwc(x), nchw_to_nhwc(k), nchw_to_nhwc(dy)
    dx = conv_dgrad_nhwc(dyn, kn, tuple(xn.shape), stride, pad)
    dk = conv_wgrad_nhwc(xn, dyn, tuple(kn.shape), stride, pad)
    return nhwc_to_nchw(dx), nhwc_to_nchw(dk)


def _bn_io(x):
    xn = nchw_to_nhwc(x)
    N, H, W, Cc = xn.shape
    return xn, N * H * W, Cc


def syncbn_forward(x, gamma, beta, eps: float, relu: bool = False):
    """syncbn_forward with group == nullptr (src/syncbn.cpp:21-70)."""
    xn, rows, Cc = _bn_io(x)
    y = torch.empty_like(xn)
    mean = torch.empty(Cc, device=x.device, dtype=torch.float32)
    invstd = torch.empty_like(mean)
    check(L().sdb_bn_fwd(ctx(), dt(x), ptr(xn), ptr(gamma), ptr(beta), ptr(y), ptr(mean), ptr(invstd), rows, Cc, eps,
                         1 if relu else 0, stream()))
    return nhwc_to_nchw(y), mean, invstd


def syncbn_backward(dy, x, mean, invstd, gamma, y_relu=None):
    """syncbn_backward with group == nullptr (src/syncbn.cpp:72-117)."""
    xn, rows, Cc = _bn_io(x)
    dyn = nchw_to_nhwc(dy.to(x.dtype))
    yr = nchw_to_nhwc(y_relu) if y_relu is not None else None
    dx = torch.empty_like(xn)
    dgamma = torch.empty(Cc, device=x.device, dtype=torch.float32)
    dbeta = torch.empty_like(dgamma)
    check(L().sdb_bn_bwd(ctx(), dt(x), ptr(dyn), ptr(xn), ptr(yr), ptr(gamma), ptr(mean), ptr(invstd), ptr(dx),
                         ptr(dgamma), ptr(dbeta), rows, Cc, stream()))
    return nhwc_to_nchw(dx), dgamma, dbeta


def syncbn_forward_group(x, gamma, beta, eps: float, relu: bool = False):
    """syncbn_forward with the context's ranks as the group (src/syncbn.cpp:21-70):
    returns (y, mean, invstd, agg) -- agg = [sum, sumsq, count] after the allreduce."""
    xn, rows, Cc = _bn_io(x)
    y = torch.empty_like(xn)
    mean = torch.empty(Cc, device=x.device, dtype=torch.float32)
    invstd = torch.empty_like(mean)
    agg = torch.empty(2 * Cc + 1, device=x.device, dtype=torch.float32)
    check(L().sdb_syncbn_fwd(ctx(), dt(x), ptr(xn), ptr(gamma), ptr(beta), ptr(y), ptr(mean), ptr(invstd), ptr(agg),
                             rows, Cc, eps, 1 if relu else 0, stream()))
    return nhwc_to_nchw(y), mean, invstd, agg


def syncbn_backward_group(dy, x, mean, invstd, gamma, agg, y_relu=None):
    """syncbn_backward with the context's ranks as the group (src/syncbn.cpp:72-117)."""
    xn, rows, Cc = _bn_io(x)
    dyn = nchw_to_nhwc(dy.to(x.dtype))
    yr = nchw_to_nhwc(y_relu) if y_relu is not None else None
    dx = torch.empty_like(xn)
    dgamma = torch.empty(Cc, device=x.device, dtype=torch.float32)
    dbeta = torch.empty_like(dgamma)
    red = torch.empty(2 * Cc, device=x.device, dtype=torch.float32)
    check(L().sdb_syncbn_bwd(ctx(), dt(x), ptr(dyn), ptr(xn), ptr(yr), ptr(gamma), ptr(mean), ptr(invstd), ptr(agg),
                             ptr(red), ptr(dx), ptr(dgamma), ptr(dbeta), rows, Cc, stream()))
    return nhwc_to_nchw(dx), dgamma, dbeta


def iabn_forward(x, gamma, beta, eps: float, slope: float):
    """iabn_forward (src/memopt.cpp:226-276): y = leaky(BN(x)); saves y only."""
    xn, rows, Cc = _bn_io(x)
    y = torch.empty_like(xn)
    mean = torch.empty(Cc, device=x.device, dtype=torch.float32)
    invstd = torch.empty_like(mean)
    check(L().sdb_iabn_fwd(ctx(), dt(x), ptr(xn), ptr(gamma), ptr(beta), ptr(y), ptr(mean), ptr(invstd), rows, Cc,
                           eps, slope, stream()))
    return nhwc_to_nchw(y), mean, invstd


def iabn_backward(dy, y, mean, invstd, gamma, beta, slope: float):
    """iabn_backward (src/memopt.cpp:278-327): recompute from the output."""
    yn, rows, Cc = _bn_io(y)
    dyn = nchw_to_nhwc(dy.to(y.dtype))
    dx = torch.empty_like(yn)
    dgamma = torch.empty(Cc, device=y.device, dtype=torch.float32)
    dbeta = torch.empty_like(dgamma)
    check(L().sdb_iabn_bwd(ctx(), dt(y), ptr(dyn), ptr(yn), ptr(gamma), ptr(beta), ptr(mean), ptr(invstd), ptr(dx),
                           ptr(dgamma), ptr(dbeta), rows, Cc, slope, stream()))
    return nhwc_to_nchw(dx), dgamma, dbeta


def has_nonfinite(g) -> bool:
    """has_nonfinite (src/trainer.cpp:78-82)."""
    flag = torch.zeros(1, device=g.device, dtype=torch.int32)
    check(L().sdb_nonfinite(ctx(), dt(g), ptr(g), g.numel(), ptr(flag), stream()))
    return bool(flag.item())


def apply_sgd(w, v, gsum, lr: float, momentum: float, denom: float, w16=None, flag=None, scale=None):
    """apply_sgd (src/trainer.cpp:86-94), in place on fp32 w and v; optional fp16 shadow.
    denom = scale * K; pass `scale` (device double) to read the live loss scale."""
    if scale is None:
        mult = denom
    else:
        mult = denom  # caller passes K when the scale is on device
    check(L().sdb_fused_sgd(ctx(), dt(gsum), ptr(gsum), ptr(w), ptr(v), ptr(w16), w.numel(), lr, momentum,
                            ptr(scale), mult, ptr(flag), stream()))


def make_anchors(H, W, stride, scales, ratios):
    """anchors [H*W*A, 4] fp32, anchor a = ratio_i * n_scales + scale_j (restated, no reference op)"""
    sc = torch.tensor(scales, dtype=torch.float32)
    ra = torch.tensor(ratios, dtype=torch.float32)
    out = torch.empty((H * W * len(scales) * len(ratios), 4), device="cuda", dtype=torch.float32)
    check(L().sdb_make_anchors(ctx(), H, W, stride, C.c_void_p(sc.data_ptr()), len(scales), C.c_void_p(ra.data_ptr()),
                               len(ratios), ptr(out), stream()))
    return out


def rpn_proposal(logits, deltas, anchors, A, pre_k, iou, post_k, img_h, img_w):
    """RPN proposal layer: logits [n, n_loc, A_pad], deltas [n, n_loc, 4*A_pad] (NHWC-flat)."""
    n, n_loc, A_pad = logits.shape
    rois = torch.empty((n, post_k, 4), device=logits.device, dtype=torch.float32)
    scores = torch.empty((n, post_k), device=logits.device, dtype=torch.float32)
    count = torch.empty(n, device=logits.device, dtype=torch.int32)
    k = min(pre_k, n_loc * A)
    order = torch.empty((n, k), device=logits.device, dtype=torch.int32)
    check(L().sdb_rpn_proposal(ctx(), dt(logits), ptr(logits), ptr(deltas), ptr(anchors), n, n_loc, A, A_pad, pre_k,
                               iou, post_k, img_h, img_w, ptr(rois), ptr(scores), ptr(count), ptr(order), stream()))
    return rois, scores, count, order


def roialign_forward(feat, rois, P, spatial_scale, sampling_ratio):
    """RoIAlign (aligned) forward, reference layout: feat [N,C,H,W] -> [R,C,P,P]."""
    fn = nchw_to_nhwc(feat)
    N, H, W, Cc = fn.shape
    R = rois.shape[0]
    out = torch.empty((R, P, P, Cc), device=feat.device, dtype=feat.dtype)
    check(L().sdb_roialign_fwd(ctx(), dt(feat), ptr(fn), N, H, W, Cc, ptr(rois), R, P, spatial_scale, sampling_ratio,
                               ptr(out), stream()))
    return nhwc_to_nchw(out)


def roialign_backward(dy, feat_shape, rois, P, spatial_scale, sampling_ratio):
    """RoIAlign backward (atomics-free gather): dy [R,C,P,P] -> dfeat [N,C,H,W]."""
    N, Cc, H, W = feat_shape
    dyn = nchw_to_nhwc(dy)
    dx = torch.empty((N, H, W, Cc), device=dy.device, dtype=dy.dtype)
    check(L().sdb_roialign_bwd(ctx(), dt(dy), ptr(dyn), N, H, W, Cc, ptr(rois), rois.shape[0], P, spatial_scale,
                               sampling_ratio, ptr(dx), stream()))
    return nhwc_to_nchw(dx)


def softmax_ce(logits, labels, grad_scale=None):
    """the reference CE op (src/model.cpp:101-151): returns (loss, dlogits)"""
    R, ncls = logits.shape
    loss = torch.zeros(1, device=logits.device, dtype=torch.float64)
    dx = torch.empty_like(logits)
    check(L().sdb_softmax_ce(ctx(), dt(logits), ptr(logits), R, ncls, ncls, ptr(labels), ptr(grad_scale), ptr(loss),
                             ptr(dx), stream()))
    return loss, dx


def update_scale(scale_dev, good_dev, flag_dev, dynamic: bool, growth_interval=2000, growth=2.0, backoff=0.5,
                 min_scale=1.0, max_scale=16777216.0):
    """update_scale (src/precision.cpp:45-56) on device-resident state."""
    check(L().sdb_update_scale(ctx(), ptr(scale_dev), ptr(good_dev), ptr(flag_dev), 1 if dynamic else 0,
                               growth_interval, growth, backoff, min_scale, max_scale, stream()))


def rpn_bce(logits, labels, A, grad_scale=None):
    """RPN objectness loss: sigmoid BCE averaged over anchors labelled 0/1.
    logits [n_loc, A_pad] (NHWC-flat), labels int8 [n_loc*A]; returns (loss, dlogits)"""
    n_loc, A_pad = logits.shape
    loss = torch.zeros(1, device=logits.device, dtype=torch.float64)
    dx = torch.zeros_like(logits)
    check(L().sdb_rpn_bce(ctx(), dt(logits), ptr(logits), n_loc, A, A_pad, ptr(labels), ptr(grad_scale), ptr(loss),
                          ptr(dx), stream()))
    return loss, dx


def rpn_smoothl1(deltas, labels, targets, A, beta, norm, grad_scale=None):
    """RPN box loss: smooth-L1 over anchors labelled 1, / norm.
    deltas [n_loc, 4*A_pad], targets fp32 [n_loc*A, 4]; returns (loss, ddeltas)"""
    n_loc, A4 = deltas.shape
    loss = torch.zeros(1, device=deltas.device, dtype=torch.float64)
    dd = torch.zeros_like(deltas)
    check(L().sdb_rpn_smoothl1(ctx(), dt(deltas), ptr(deltas), n_loc, A, A4 // 4, ptr(labels), ptr(targets), beta,
                               norm, ptr(grad_scale), ptr(loss), ptr(dd), stream()))
    return loss, dd


def smoothl1(pred, labels, targets, beta, grad_scale=None):
    """RCNN class-specific box loss: pred [R, ld] (slot 4*label), targets [R, 4];
    summed over foreground RoIs, / #RoIs with label >= 0; returns (loss, dpred)"""
    R, ld = pred.shape
    loss = torch.zeros(1, device=pred.device, dtype=torch.float64)
    dp = torch.zeros_like(pred)
    check(L().sdb_smoothl1(ctx(), dt(pred), ptr(pred), R, ld, ptr(labels), ptr(targets), beta, ptr(grad_scale),
                           ptr(loss), ptr(dp), stream()))
    return loss, dp


def anchor_targets(anchors, gt, gt_count, keys, img_h, img_w, fg_thr=0.7, bg_thr=0.3, batch=256, fg_frac=0.5):
    """RPN anchor targets: anchors [nA,4], gt [n_img, G, 4], gt_count int32 [n_img],
    keys uint64 [n_img] (as int64 tensor); returns (labels int8 [n_img, nA], targets [n_img, nA, 4])"""
    nA = anchors.shape[0]
    n_img, G, _ = gt.shape
    labels = torch.empty((n_img, nA), device=anchors.device, dtype=torch.int8)
    targets = torch.empty((n_img, nA, 4), device=anchors.device, dtype=torch.float32)
    check(L().sdb_anchor_targets(ctx(), ptr(anchors), nA, n_img, ptr(gt), G, ptr(gt_count), img_h, img_w, ptr(keys),
                                 fg_thr, bg_thr, batch, fg_frac, ptr(labels), ptr(targets), stream()))
    return labels, targets


def proposal_targets(proposals, prop_count, gt, gt_cls, gt_count, keys, batch=512, fg_frac=0.25, fg_thr=0.5,
                     bg_hi=0.5, bg_lo=0.0):
    """RCNN proposal targets: proposals [n_img, P, 4], counts int32 [n_img];
    returns (rois [n_img*batch, 5], labels int32, targets [.., 4], count int32 [n_img])"""
    n_img, Pst, _ = proposals.shape
    G = gt.shape[1]
    dev = proposals.device
    rois = torch.empty((n_img * batch, 5), device=dev, dtype=torch.float32)
    labels = torch.empty(n_img * batch, device=dev, dtype=torch.int32)
    targets = torch.empty((n_img * batch, 4), device=dev, dtype=torch.float32)
    count = torch.empty(n_img, device=dev, dtype=torch.int32)
    check(L().sdb_proposal_targets(ctx(), ptr(proposals), Pst, ptr(prop_count), ptr(gt), ptr(gt_cls), G,
                                   ptr(gt_count), n_img, ptr(keys), fg_thr, bg_hi, bg_lo, batch, fg_frac, ptr(rois),
                                   ptr(labels), ptr(targets), ptr(count), stream()))
    return rois, labels, targets, count


def allreduce_sum(buf, context=None):
    """CommGroup::allreduce_sum (src/comm.cpp:288-315): in-place SUM over the
    context's ranks (NCCL); identity on a context without a communicator"""
    code = {torch.float32: F32, torch.float16: F16, torch.float64: 2}[buf.dtype]
    check(L().sdb_allreduce_sum(context if context is not None else ctx(), code, ptr(buf), buf.numel(), stream()))
    return buf
