"""GPU parity: libsdb conv / BN / IABN / optimizer kernels vs the compiled
reference engine (oracle/_ref) on identical seeded inputs.  Runs through the
C ABI (paper_1903_05831_b200.simdet mirrors the reference signatures)."""
import numpy as np
import pytest

import oracle
from tests.util import assert_close

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CONV_CASES = [
    # (N, C, H, W, K, R, S, stride, pad)
    (2, 16, 12, 10, 32, 3, 3, 1, 1),
    (2, 64, 9, 11, 64, 1, 1, 1, 0),
    (2, 32, 10, 10, 64, 1, 1, 2, 0),
    (2, 8, 32, 32, 64, 7, 7, 2, 3),
    (1, 16, 9, 9, 16, 3, 3, 2, 1),
    (1, 24, 7, 5, 40, 3, 3, 1, 1),
    (2, 64, 20, 24, 256, 3, 3, 1, 1),
    (1, 3, 11, 13, 8, 3, 3, 1, 1),
    # all-TMA path (C % 64 == 0 / K % 64 == 0): im2col boxes that wrap rows and
    # images, stride 2, sub-pixel dgrad phases, BN = 64/128/256, split-K wgrad
    (2, 128, 15, 13, 128, 3, 3, 2, 1),
    (3, 64, 14, 14, 128, 1, 1, 2, 0),
    (2, 256, 10, 9, 512, 1, 1, 1, 0),
    (1, 192, 7, 7, 64, 3, 3, 1, 1),
    (2, 64, 30, 31, 64, 3, 3, 1, 1),
    (4, 128, 28, 28, 256, 3, 3, 1, 1),
]


def _rand(rng, shape, fp16, scale=1.0):
    a = (rng.standard_normal(shape) * scale).astype(np.float32)
    if fp16:
        a = a.astype(np.float16).astype(np.float32)
    return a


def _ref_conv(x, k, stride, pad, fp16):
    N, C, H, W = x.shape
    O, _, kh, kw = k.shape
    Ho, Wo = (H + 2 * pad - kh) // stride + 1, (W + 2 * pad - kw) // stride + 1
    y = np.zeros((N, O, Ho, Wo), np.float32)
    rc = oracle.ref().ref_conv2d(oracle.p(x), N, C, H, W, oracle.p(k), O, kh, kw, stride, pad, int(fp16), oracle.p(y))
    assert rc == 0
    return y


def _ref_conv_bwd(x, k, dy, stride, pad, fp16):
    N, C, H, W = x.shape
    O, _, kh, kw = k.shape
    dx = np.zeros_like(x)
    dk = np.zeros_like(k)
    rc = oracle.ref().ref_conv2d_backward(oracle.p(x), N, C, H, W, oracle.p(k), O, kh, kw, stride, pad, int(fp16),
                                          oracle.p(dy), oracle.p(dx), oracle.p(dk))
    assert rc == 0
    return dx, dk


@pytest.mark.parametrize("fp16", [False, True])
@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_fwd_bwd(ref, case, fp16):
    from paper_1903_05831_b200 import simdet as sd
    N, C, H, W, K, R, S, st, pd = case
    rng = np.random.default_rng(hash(case) % 2**32)
    x = _rand(rng, (N, C, H, W), fp16)
    k = _rand(rng, (K, C, R, S), fp16, 1.0 / np.sqrt(C * R * S))
    y_ref = _ref_conv(x, k, st, pd, fp16)
    dy = _rand(rng, y_ref.shape, fp16)
    dx_ref, dk_ref = _ref_conv_bwd(x, k, dy, st, pd, fp16)
    tdt = torch.float16 if fp16 else torch.float32
    xt, kt, dyt = (torch.from_numpy(a).to("cuda", tdt) for a in (x, k, dy))
    y = sd.conv2d(xt, kt, st, pd)
    dx, dk = sd.conv2d_backward(xt, kt, dyt, st, pd)
    torch.cuda.synchronize()
    tol = 2e-3 if fp16 else 1e-5
    assert_close(y, y_ref, tol, "y")
    assert_close(dx, dx_ref, tol, "dx")
    assert_close(dk, dk_ref, tol, "dk")


def test_conv_large_tile_path(ref):
    """exercises the 128x256 tensor-core tile (enough tiles to pick BN=256)."""
    from paper_1903_05831_b200 import simdet as sd
    rng = np.random.default_rng(7)
    N, C, H, W, K = 8, 64, 56, 56, 512
    x = _rand(rng, (N, C, H, W), True)
    k = _rand(rng, (K, C, 1, 1), True, 0.125)
    y_ref = _ref_conv(x, k, 1, 0, True)
    y = sd.conv2d(torch.from_numpy(x).cuda().half(), torch.from_numpy(k).cuda().half(), 1, 0)
    assert_close(y, y_ref, 2e-3, "y")


# small-M layers whose 128x256 tiles fill less than half the SMs (the
# narrow-tile choice); odd k-block counts and partial M tiles included
SMALL_M_CASES = [(2, 256, 50, 84, 256, 3, 3, 1, 1), (2, 1024, 50, 84, 256, 1, 1, 1, 0), (2, 256, 50, 84, 1024, 1, 1, 1, 0),
                (1, 192, 13, 17, 256, 3, 3, 1, 1)]


@pytest.mark.parametrize("case", SMALL_M_CASES)
def test_conv_small_m_layers(case):
    """fprop and dgrad of the res4-sized layers vs an fp32 torch reference"""
    from paper_1903_05831_b200 import simdet as sd
    N, C, H, W, K, R, S, st, pd = case
    g = torch.Generator(device="cuda").manual_seed(hash(case) % 2**31)
    x = torch.randn((N, H, W, C), device="cuda", generator=g).half()
    w = (torch.randn((K, R, S, C), device="cuda", generator=g) / np.sqrt(C * R * S)).half()
    y = sd.conv_fprop_nhwc(x, w, st, pd)
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2), stride=st,
                                     padding=pd).permute(0, 2, 3, 1)
    dy = torch.randn(ref.shape, device="cuda", generator=g).half()
    dx = sd.conv_dgrad_nhwc(dy, w, (N, H, W, C), st, pd)
    dref = torch.nn.grad.conv2d_input((N, C, H, W), w.float().permute(0, 3, 1, 2), dy.float().permute(0, 3, 1, 2),
                                      stride=st, padding=pd).permute(0, 2, 3, 1)
    y2 = sd.conv_fprop_nhwc(x, w, st, pd)
    torch.cuda.synchronize()
    assert_close(y.float(), ref, 2e-3, "y")
    assert_close(dx.float(), dref, 2e-3, "dx")
    assert torch.equal(y, y2), "conv must be deterministic"


# (N, H, W, C, K, R, S, stride, pad): the first four take the TMA residual
# epilogue (stride 1, BN = 256, sign bitmap), the last two fall back to the
# fp16-mask epilogue (BN = 128 / stride 2) and must ignore the bitmap
DGRAD_ACT_CASES = [(2, 20, 30, 256, 64, 1, 1, 1, 0), (16, 7, 7, 2048, 512, 1, 1, 1, 0), (1, 25, 42, 1024, 256, 3, 3, 1, 1),
                   (2, 13, 17, 512, 128, 1, 1, 1, 0), (2, 9, 9, 128, 64, 1, 1, 1, 0), (2, 14, 14, 256, 128, 3, 3, 2, 1)]


@pytest.mark.parametrize("case", DGRAD_ACT_CASES)
def test_dgrad_act_bitmap_matches_fp16_mask(case):
    """the step's fused residual + leaky backward: the sign-bitmap epilogue is
    bit-identical to the fp16-mask one, and both match an fp32 torch reference"""
    from paper_1903_05831_b200 import simdet as sd
    N, H, W, C, K, R, S, st, pd = case
    g = torch.Generator(device="cuda").manual_seed(hash(case) % 2**31)
    Ho, Wo = (H + 2 * pd - R) // st + 1, (W + 2 * pd - S) // st + 1
    dy = torch.randn((N, Ho, Wo, K), device="cuda", generator=g).half()
    w = (torch.randn((K, R, S, C), device="cuda", generator=g) / np.sqrt(K * R * S)).half()
    add = torch.randn((N, H, W, C), device="cuda", generator=g).half()
    y = torch.randn((N, H, W, C), device="cuda", generator=g).half()
    y[..., ::7] = 0  # y == 0 takes the negative branch
    neg = 0.01
    bits = sd.sign_bits_nhwc(y)
    dx_m = sd.conv_dgrad_act_nhwc(dy, w, add, y, neg, st, pd)
    dx_b = sd.conv_dgrad_act_nhwc(dy, w, add, y, neg, st, pd, y_bits=bits)
    torch.cuda.synchronize()
    assert torch.equal(dx_m.view(torch.int16), dx_b.view(torch.int16))
    # fp32 reference of the same op
    acc = torch.nn.grad.conv2d_input((N, C, H, W), w.float().permute(0, 3, 1, 2), dy.float().permute(0, 3, 1, 2),
                                     stride=st, padding=pd).permute(0, 2, 3, 1)
    p = (acc + add.float()).half().float()
    ref = torch.where(y.float() > 0, p, (p * neg).half().float())
    assert_close(dx_m.float(), ref, 2e-3, "dx")


# the last two are large enough that every CTA of the bulk-copy statistics
# pipeline streams more tiles than it has stages (ring wrap-around)
BN_SHAPES = [(2, 64, 7, 9), (4, 256, 5, 5), (2, 2048, 3, 3), (1, 8, 4, 4), (2, 512, 16, 12), (6, 128, 150, 160),
             (2, 1024, 41, 37)]


@pytest.mark.parametrize("fp16", [False, True])
@pytest.mark.parametrize("shape", BN_SHAPES)
def test_bn_fwd_bwd(ref, shape, fp16):
    from paper_1903_05831_b200 import simdet as sd
    N, C, H, W = shape
    rng = np.random.default_rng(C + H)
    x = _rand(rng, shape, fp16, 2.0) + 0.5
    x = x.astype(np.float16).astype(np.float32) if fp16 else x
    g = (1.0 + 0.2 * rng.standard_normal(C)).astype(np.float32)
    b = (0.1 * rng.standard_normal(C)).astype(np.float32)
    y_ref = np.zeros_like(x)
    mean_ref = np.zeros(C, np.float32)
    inv_ref = np.zeros(C, np.float32)
    assert ref.ref_bn_forward(oracle.p(x), N, C, H, W, oracle.p(g), oracle.p(b), 1e-5, int(fp16), oracle.p(y_ref),
                              oracle.p(mean_ref), oracle.p(inv_ref)) == 0
    dy = _rand(rng, shape, fp16)
    dx_ref = np.zeros_like(x)
    dg_ref = np.zeros(C, np.float32)
    db_ref = np.zeros(C, np.float32)
    assert ref.ref_bn_backward(oracle.p(dy), oracle.p(x), N, C, H, W, oracle.p(g), oracle.p(mean_ref),
                               oracle.p(inv_ref), int(fp16), oracle.p(dx_ref), oracle.p(dg_ref), oracle.p(db_ref)) == 0
    tdt = torch.float16 if fp16 else torch.float32
    xt = torch.from_numpy(x).to("cuda", tdt)
    gt, bt = torch.from_numpy(g).cuda(), torch.from_numpy(b).cuda()
    y, mean, inv = sd.syncbn_forward(xt, gt, bt, 1e-5)
    dx, dg, db = sd.syncbn_backward(torch.from_numpy(dy).to("cuda", tdt), xt, mean, inv, gt)
    torch.cuda.synchronize()
    tol = 1e-2 if fp16 else 1e-3
    assert_close(mean, mean_ref, 1e-5, "mean")
    assert_close(inv, inv_ref, 1e-5, "invstd")
    assert_close(y, y_ref, tol, "y")
    assert_close(dx, dx_ref, tol, "dx")
    assert_close(dg, dg_ref, tol, "dgamma")
    assert_close(db, db_ref, tol, "dbeta")


@pytest.mark.parametrize("fp16", [False, True])
@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("shape", [(2, 64, 7, 9), (6, 128, 150, 160)])
def test_syncbn_group_world1(ref, shape, fp16, relu):
    """SyncBN through the context's group (sdb_syncbn_fwd/bwd: local sums, NCCL
    allreduce -- the identity at one rank --, global statistics) is bit-identical
    to plain BN at world 1; its reduction buffer holds the reference's
    [sum, sumsq, count] (K = 1 run_workers group)"""
    from paper_1903_05831_b200 import simdet as sd
    N, C, H, W = shape
    rng = np.random.default_rng(C + H + 7)
    x = _rand(rng, shape, fp16, 2.0) + 0.5
    x = x.astype(np.float16).astype(np.float32) if fp16 else x
    g = (1.0 + 0.2 * rng.standard_normal(C)).astype(np.float32)
    b = (0.1 * rng.standard_normal(C)).astype(np.float32)
    dy = _rand(rng, shape, fp16)
    tdt = torch.float16 if fp16 else torch.float32
    xt, dyt = torch.from_numpy(x).to("cuda", tdt), torch.from_numpy(dy).to("cuda", tdt)
    gt, bt = torch.from_numpy(g).cuda(), torch.from_numpy(b).cuda()
    y0, m0, i0 = sd.syncbn_forward(xt, gt, bt, 1e-5, relu=relu)
    y1, m1, i1, agg = sd.syncbn_forward_group(xt, gt, bt, 1e-5, relu=relu)
    dx0, dg0, db0 = sd.syncbn_backward(dyt, xt, m0, i0, gt, y_relu=y0 if relu else None)
    dx1, dg1, db1 = sd.syncbn_backward_group(dyt, xt, m1, i1, gt, agg, y_relu=y1 if relu else None)
    torch.cuda.synchronize()
    for a0, a1 in ((y0, y1), (m0, m1), (i0, i1), (dx0, dx1), (dg0, dg1), (db0, db1)):
        assert torch.equal(a0, a1)
    y_r = np.zeros((1,) + shape, np.float32)
    m_r, i_r = np.zeros(C, np.float32), np.zeros(C, np.float32)
    agg_r = np.zeros(2 * C + 1, np.float32)
    assert ref.ref_syncbn_forward_k(1, oracle.p(x), N, C, H, W, oracle.p(g), oracle.p(b), 1e-5, int(fp16),
                                    oracle.p(y_r), oracle.p(m_r), oracle.p(i_r), oracle.p(agg_r)) == 0
    a = agg.cpu().numpy()
    assert a[2 * C] == agg_r[2 * C] == N * H * W
    assert_close(a[:2 * C], agg_r[:2 * C], 1e-6, "local sums")
    assert_close(m1, m_r, 1e-5, "mean")


@pytest.mark.parametrize("fp16", [False, True])
@pytest.mark.parametrize("slope", [0.1, 1.0])
@pytest.mark.parametrize("shape", BN_SHAPES)
def test_iabn_fwd_bwd(ref, shape, fp16, slope):
    from paper_1903_05831_b200 import simdet as sd
    N, C, H, W = shape
    rng = np.random.default_rng(3 * C + W)
    x = _rand(rng, shape, fp16, 1.5) - 0.25
    x = x.astype(np.float16).astype(np.float32) if fp16 else x
    g = (1.0 + 0.2 * rng.standard_normal(C)).astype(np.float32)
    g[np.abs(g) < 0.05] = 0.5
    b = (0.1 * rng.standard_normal(C)).astype(np.float32)
    y_ref = np.zeros_like(x)
    mean_ref = np.zeros(C, np.float32)
    inv_ref = np.zeros(C, np.float32)
    assert ref.ref_iabn_forward(oracle.p(x), N, C, H, W, oracle.p(g), oracle.p(b), 1e-5, slope, int(fp16),
                                oracle.p(y_ref), oracle.p(mean_ref), oracle.p(inv_ref)) == 0
    dy = _rand(rng, shape, fp16)
    dx_ref = np.zeros_like(x)
    dg_ref = np.zeros(C, np.float32)
    db_ref = np.zeros(C, np.float32)
    assert ref.ref_iabn_backward(oracle.p(dy), oracle.p(y_ref), N, C, H, W, oracle.p(g), oracle.p(b),
                                 oracle.p(mean_ref), oracle.p(inv_ref), 1e-5, slope, int(fp16), oracle.p(dx_ref),
                                 oracle.p(dg_ref), oracle.p(db_ref)) == 0
    tdt = torch.float16 if fp16 else torch.float32
    gt, bt = torch.from_numpy(g).cuda(), torch.from_numpy(b).cuda()
    y, mean, inv = sd.iabn_forward(torch.from_numpy(x).to("cuda", tdt), gt, bt, 1e-5, slope)
    dx, dg, db = sd.iabn_backward(torch.from_numpy(dy).to("cuda", tdt), y, mean, inv, gt, bt, slope)
    torch.cuda.synchronize()
    tol = 1e-2 if fp16 else 1e-3
    assert_close(y, y_ref, tol, "y")
    assert_close(dx, dx_ref, tol, "dx")
    assert_close(dg, dg_ref, tol, "dgamma")
    assert_close(db, db_ref, tol, "dbeta")


def test_iabn_errors():
    """NonInvertibleError / DegenerateBatchError, src/memopt.cpp:229-235."""
    import paper_1903_05831_b200 as pkg
    from paper_1903_05831_b200 import simdet as sd
    x = torch.randn(2, 8, 3, 3, device="cuda")
    g = torch.ones(8, device="cuda")
    b = torch.zeros(8, device="cuda")
    with pytest.raises(pkg.NonInvertibleError):
        sd.iabn_forward(x, g, b, 1e-5, 0.0)
    g0 = g.clone()
    g0[3] = 0
    with pytest.raises(pkg.NonInvertibleError):
        sd.iabn_forward(x, g0, b, 1e-5, 0.1)
    with pytest.raises(pkg.DegenerateBatchError):
        sd.iabn_forward(torch.randn(1, 8, 1, 1, device="cuda"), g, b, 1e-5, 0.1)


@pytest.mark.parametrize("gfp16", [False, True])
@pytest.mark.parametrize("n", [1 << 20 | 77, 1 << 20])  # scalar tail path / 8-wide vector path
def test_fused_sgd_bitwise(orc, gfp16, n):
    """apply_sgd (src/trainer.cpp:86-94) is FP32 elementwise: compare bit for bit."""
    from paper_1903_05831_b200 import simdet as sd
    rng = np.random.default_rng(11)
    w = rng.standard_normal(n).astype(np.float32)
    v = (0.01 * rng.standard_normal(n)).astype(np.float32)
    g = (300 * rng.standard_normal(n)).astype(np.float32)
    if gfp16:
        g = g.astype(np.float16).astype(np.float32)
    scale, K = 128.0, 4
    w_o, v_o = w.copy(), v.copy()
    orc.orc_apply_sgd(oracle.p(w_o), oracle.p(v_o), oracle.p(g), n, 0.01, 0.9, scale * K)
    wt, vt = torch.from_numpy(w).cuda(), torch.from_numpy(v).cuda()
    gt = torch.from_numpy(g).cuda().to(torch.float16 if gfp16 else torch.float32)
    w16 = torch.empty(n, device="cuda", dtype=torch.float16)
    sc = torch.tensor([scale], dtype=torch.float64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    sd.apply_sgd(wt, vt, gt, 0.01, 0.9, float(K), w16=w16, flag=flag, scale=sc)
    torch.cuda.synchronize()
    assert np.array_equal(wt.cpu().numpy().view(np.uint32), w_o.view(np.uint32))
    assert np.array_equal(vt.cpu().numpy().view(np.uint32), v_o.view(np.uint32))
    assert np.array_equal(w16.cpu().numpy(), w_o.astype(np.float16))
    # overflow flag set -> untouched (src/trainer.cpp:253)
    flag.fill_(1)
    before = wt.clone()
    sd.apply_sgd(wt, vt, gt, 0.01, 0.9, float(K), flag=flag, scale=sc)
    torch.cuda.synchronize()
    assert torch.equal(before, wt)


def test_nonfinite():
    from paper_1903_05831_b200 import simdet as sd
    for dtp in (torch.float32, torch.float16):
        g = torch.randn(100003, device="cuda").to(dtp)
        assert not sd.has_nonfinite(g)
        g[77777] = float("inf")
        assert sd.has_nonfinite(g)
        g[77777] = float("nan")
        assert sd.has_nonfinite(g)


def test_update_scale_matches_reference(ref):
    """device update_scale vs the reference's (src/precision.cpp:45-56)."""
    from paper_1903_05831_b200 import simdet as sd
    import ctypes as C
    rng = np.random.default_rng(5)
    pattern = (rng.random(400) < 0.1).astype(np.int32)
    s_ref, g_ref = C.c_double(32768.0), C.c_int64(0)
    sc = torch.tensor([32768.0], dtype=torch.float64, device="cuda")
    good = torch.zeros(1, dtype=torch.int64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    for ov in pattern:
        ref.ref_update_scale(C.byref(s_ref), C.byref(g_ref), 1, 7, 2.0, 0.5, 1.0, 2.0**24, int(ov))
        flag.fill_(int(ov))
        sd.update_scale(sc, good, flag, True, growth_interval=7)
        torch.cuda.synchronize()
        assert sc.item() == s_ref.value and good.item() == g_ref.value


@pytest.mark.parametrize("case", [
    # (N, H, W, C, K, R, stride): tile widths 256 / 128 / 64 on the TMA-store path, M % 128 != 0
    (2, 60, 61, 64, 512, 1, 1),    # BN = 256 (res5-like expansion width), M = 7320
    (2, 47, 33, 128, 128, 3, 1),   # BN = 128, 3x3, M = 3102
    (1, 29, 43, 64, 64, 1, 1),     # BN = 64, M = 1247
    (2, 30, 31, 256, 1024, 1, 2),  # stride-2 1x1 into 1024 channels (res4 down), M = 480
])
@pytest.mark.parametrize("iabn", [False, True])
def test_fused_norm_statistics_in_fprop_epilogue(case, iabn):
    """the fp64 column sums reduced in the fprop's TMA-store epilogue
    (ConvStats -> finalize) give the same mean/invstd as the separate statistics
    pass over the same fp16 output, for every tile width and ragged M"""
    from paper_1903_05831_b200 import simdet as sd
    N, H, W, C, K, R, s = case
    pad = R // 2
    g = torch.Generator(device="cuda").manual_seed(sum(case))
    x = (torch.randn((N, H, W, C), generator=g, device="cuda") * 2 + 0.5).half()
    w = (torch.randn((K, R, R, C), generator=g, device="cuda") * (1.0 / (C * R * R) ** 0.5)).half()
    y, mean, invstd, fused = sd.conv_fprop_stats_nhwc(x, w, s, pad, iabn=iabn)
    assert fused, "the fused-statistics epilogue did not run for this shape"
    rows = y.shape[0] * y.shape[1] * y.shape[2]
    gm = torch.ones(K, device="cuda")
    bt = torch.zeros(K, device="cuda")
    m2, i2 = torch.empty_like(mean), torch.empty_like(invstd)
    out = torch.empty_like(y)
    if iabn:
        sd.check(sd.L().sdb_iabn_fwd(sd.ctx(), 1, sd.ptr(y), sd.ptr(gm), sd.ptr(bt), sd.ptr(out), sd.ptr(m2), sd.ptr(i2),
                                     rows, K, 1e-5, 1.0, sd.stream()))
    else:
        sd.check(sd.L().sdb_bn_fwd(sd.ctx(), 1, sd.ptr(y), sd.ptr(gm), sd.ptr(bt), sd.ptr(out), sd.ptr(m2), sd.ptr(i2),
                                   rows, K, 1e-5, 0, sd.stream()))
    torch.cuda.synchronize()
    # both reduce the same fp16 values in fp64; only the summation order differs
    assert torch.allclose(mean, m2, rtol=1e-6, atol=1e-7), (mean - m2).abs().max()
    assert torch.allclose(invstd, i2, rtol=1e-6), (invstd - i2).abs().max()
    # and against a float64 recomputation from y
    yd = y.double().reshape(-1, K)
    mu = yd.mean(0)
    var = (yd * yd).mean(0) - mu * mu
    assert torch.allclose(mean.double(), mu, rtol=1e-5, atol=1e-6)
    assert torch.allclose(invstd.double(), 1.0 / torch.sqrt(var.clamp_min(0) + 1e-5), rtol=1e-4)


@pytest.mark.parametrize("case,expect_fused", [
    # (N, H, W, C = IABN channels = dgrad output, K = conv output channels, R): dgrad tile widths 256 / 128 / 64
    ((256, 7, 7, 512, 2048, 1), False),  # res5 conv3-like, BN = 256: unfused by design (stats pass)
    ((2, 50, 84, 256, 1024, 1), True),   # res4 conv3: BN = 128 (narrow rule), M = 8400
    ((2, 47, 33, 128, 128, 3), True),    # res3 conv2-like 3x3: BN = 128, ragged M = 3102
    ((1, 63, 41, 64, 256, 1), True),     # res2 conv3-like: BN = 64, ragged M = 2583
    ((2, 40, 37, 64, 64, 3), True),      # res2 conv2-like 3x3: BN = 64
])
def test_dgrad_fused_iabn_backward_statistics(ref, case, expect_fused):
    """The InPlace-ABN backward sums reduced in the dgrad epilogue (y by TMA next
    to the staged dy box) give the same dgamma/dbeta/dz as the separate
    statistics pass over the same tensors; the dgrad output itself is bitwise
    the plain dgrad; and both agree with the reference iabn_backward"""
    from paper_1903_05831_b200 import simdet as sd
    N, H, W, Cc, K, R = case
    pad = R // 2
    g = torch.Generator(device="cuda").manual_seed(sum(case))
    # y: a stored IABN output (leaky 0.1 of N(beta, gamma)), dy: the conv's output gradient
    gamma = (torch.rand(Cc, generator=g, device="cuda") + 0.5)
    beta = (torch.rand(Cc, generator=g, device="cuda") - 0.5) * 0.4
    xh = torch.randn((N, H, W, Cc), generator=g, device="cuda")
    yv = xh * gamma + beta
    y = torch.where(yv >= 0, yv, 0.1 * yv).half()
    invstd = (torch.rand(Cc, generator=g, device="cuda") + 0.5)
    dy = torch.randn((N, H, W, K), generator=g, device="cuda").half()
    w = (torch.randn((K, R, R, Cc), generator=g, device="cuda") * (1.0 / (K * R * R) ** 0.5)).half()
    dyi, dz, dgm, dbt, fused = sd.conv_dgrad_iabn_bwd_nhwc(dy, w, y, gamma, beta, invstd, 0.1, pad)
    assert fused == expect_fused, "which statistics path ran"
    # unfused: plain dgrad, then the IABN backward statistics pass
    dyi2 = sd.conv_dgrad_nhwc(dy, w, (N, H, W, Cc), 1, pad)
    rows = N * H * W
    dz2 = torch.empty_like(dz)
    dgm2, dbt2 = torch.empty_like(dgm), torch.empty_like(dbt)
    sd.check(sd.L().sdb_iabn_bwd(sd.ctx(), 1, sd.ptr(dyi2), sd.ptr(y), sd.ptr(gamma), sd.ptr(beta), None,
                                 sd.ptr(invstd), sd.ptr(dz2), sd.ptr(dgm2), sd.ptr(dbt2), rows, Cc, 0.1, sd.stream()))
    torch.cuda.synchronize()
    assert torch.equal(dyi, dyi2), "the dgrad output must not depend on the epilogue variant"
    # same fp64 sums in another order: float results agree to the last bits
    assert torch.allclose(dgm, dgm2, rtol=1e-6, atol=1e-5), (dgm - dgm2).abs().max()
    assert torch.allclose(dbt, dbt2, rtol=1e-6, atol=1e-5), (dbt - dbt2).abs().max()
    assert (dz.float() - dz2.float()).abs().max() <= 2e-3 * dz2.float().abs().max()
    # the reference iabn_backward on the same (NCHW) tensors
    ynp = np.ascontiguousarray(y.float().permute(0, 3, 1, 2).cpu().numpy())
    dnp = np.ascontiguousarray(dyi.float().permute(0, 3, 1, 2).cpu().numpy())
    dx_r = np.zeros_like(ynp)
    dg_r, db_r = np.zeros(Cc, np.float32), np.zeros(Cc, np.float32)
    gn, bn_, isn = (gamma.cpu().numpy(), beta.cpu().numpy(), invstd.cpu().numpy())
    mean0 = np.zeros(Cc, np.float32)
    assert ref.ref_iabn_backward(oracle.p(dnp), oracle.p(ynp), N, Cc, H, W, oracle.p(gn), oracle.p(bn_),
                                 oracle.p(mean0), oracle.p(isn), 1e-5, 0.1, 1, oracle.p(dx_r), oracle.p(dg_r),
                                 oracle.p(db_r)) == 0
    assert_close(dgm, dg_r, 1e-5, "dgamma vs reference")
    assert_close(dbt, db_r, 1e-5, "dbeta vs reference")
    assert_close(dz.float().permute(0, 3, 1, 2), dx_r, 1e-2, "dz vs reference")
