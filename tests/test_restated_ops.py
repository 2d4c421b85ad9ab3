"""Known-answer and independent cross-checks for the CPU restatement of the
operators the reference does not implement (oracle/restate.cpp) -- "parity
unpinned by the reference", so pinned here: hand-computed values and
torch / torchvision as independent implementations of the same semantics."""
import math

import numpy as np
import pytest

import oracle
from oracle import p

torch = pytest.importorskip("torch")


def test_expf_is_accurate(orc):
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(-20, 20, 5000), rng.uniform(-87, 88, 1000), [0.0, 1.0, -1.0, 4.135]])
    for x in xs.astype(np.float32):
        got = np.float32(orc.orc_expf(float(x)))
        want = np.float32(math.exp(float(x)))
        ulp = abs(int(got.view(np.int32)) - int(want.view(np.int32)))
        assert ulp <= 1, (x, got, want)


def test_anchor_known_answer(orc):
    out = np.zeros((1, 4), np.float32)
    s, r = np.array([32.0], np.float32), np.array([1.0], np.float32)
    orc.orc_anchors(1, 1, 16.0, p(s), 1, p(r), 1, p(out))
    assert out.tolist() == [[-8.0, -8.0, 24.0, 24.0]]
    # ratio 2 (h/w): w = 32/sqrt2, h = 32*sqrt2; anchor a = i*ns + j
    s = np.array([32.0, 64.0, 128.0], np.float32)
    r = np.array([0.5, 2.0], np.float32)
    out = np.zeros((2 * 6, 4), np.float32)
    orc.orc_anchors(1, 2, 16.0, p(s), 3, p(r), 2, p(out))
    a = out.reshape(2, 2, 3, 4)  # (x, ratio, scale)
    w = a[..., 2] - a[..., 0]
    h = a[..., 3] - a[..., 1]
    np.testing.assert_allclose(h / w, np.array([0.5, 2.0])[None, :, None] * np.ones((2, 2, 3)), rtol=1e-6)
    np.testing.assert_allclose(np.sqrt(w * h)[0, 0], [32, 64, 128], rtol=1e-6)
    assert np.allclose((a[1, ..., 0] + a[1, ..., 2]) / 2, 24.0)


def test_decode_encode_roundtrip(orc):
    rng = np.random.default_rng(1)
    n = 500
    xy = rng.uniform(30, 500, (n, 2))  # keep the GT inside the clip window
    wh = rng.uniform(8, 200, (n, 2))
    ex = np.concatenate([xy, xy + wh], 1).astype(np.float32)
    gxy = xy + rng.uniform(-20, 20, (n, 2))
    gwh = wh * np.exp(rng.uniform(-0.5, 0.5, (n, 2)))
    gt = np.concatenate([gxy, gxy + gwh], 1).astype(np.float32)
    w = np.array([1, 1, 1, 1], np.float32)
    t = np.zeros_like(ex)
    orc.orc_encode(p(ex), p(gt), n, p(w), p(t))
    back = np.zeros_like(ex)
    orc.orc_decode(p(ex), p(t), n, p(w), 100.0, 1e9, 1e9, p(back))
    np.testing.assert_allclose(back, gt, rtol=1e-4, atol=1e-2)


def test_roialign_matches_torchvision(orc):
    tv = pytest.importorskip("torchvision")
    rng = np.random.default_rng(2)
    N, C, H, W, P = 2, 5, 13, 17, 7
    feat = rng.standard_normal((N, C, H, W)).astype(np.float32)
    R = 40
    b = rng.integers(0, N, R)
    x1 = rng.uniform(-40, 17 * 16, R)
    y1 = rng.uniform(-40, 13 * 16, R)
    rois = np.stack([b, x1, y1, x1 + rng.uniform(1, 200, R), y1 + rng.uniform(1, 150, R)], 1).astype(np.float32)
    out = np.zeros((R, C, P, P), np.float32)
    orc.orc_roialign_fwd(p(feat), N, C, H, W, p(rois), R, P, 1 / 16, 2, 1, p(out))
    ft = torch.from_numpy(feat).requires_grad_(True)
    ref = tv.ops.roi_align(ft, torch.from_numpy(rois), (P, P), spatial_scale=1 / 16, sampling_ratio=2, aligned=True)
    np.testing.assert_allclose(out, ref.detach().numpy(), rtol=1e-5, atol=1e-5)
    dy = rng.standard_normal(out.shape).astype(np.float32)
    ref.backward(torch.from_numpy(dy))
    dfeat = np.zeros_like(feat)
    orc.orc_roialign_bwd(p(dy), N, C, H, W, p(rois), R, P, 1 / 16, 2, 1, p(dfeat))
    np.testing.assert_allclose(dfeat, ft.grad.numpy(), rtol=1e-4, atol=1e-4)


def test_roialign_hand_value(orc):
    # 1 channel 2x2 feature [[0,1],[2,3]], RoI covering it exactly (aligned: corners at
    # pixel edges), P=1, sr=1 -> sample at the centre (0.5,0.5) -> mean 1.5
    feat = np.array([[[[0.0, 1.0], [2.0, 3.0]]]], np.float32)
    rois = np.array([[0, 0, 0, 2, 2]], np.float32)
    out = np.zeros((1, 1, 1, 1), np.float32)
    orc.orc_roialign_fwd(p(feat), 1, 1, 2, 2, p(rois), 1, 1, 1.0, 1, 1, p(out))
    assert out[0, 0, 0, 0] == 1.5


def test_maxpool_matches_torch(orc):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 3, 11, 9)).astype(np.float32)
    y = np.zeros((2, 3, 6, 5), np.float32)
    orc.orc_maxpool_fwd(p(x), 2, 3, 11, 9, 3, 2, 1, p(y))
    xt = torch.from_numpy(x).requires_grad_(True)
    yt = torch.nn.functional.max_pool2d(xt, 3, 2, 1)
    assert np.array_equal(y, yt.detach().numpy())
    dy = rng.standard_normal(y.shape).astype(np.float32)
    yt.backward(torch.from_numpy(dy))
    dx = np.zeros_like(x)
    orc.orc_maxpool_bwd(p(x), p(dy), 2, 3, 11, 9, 3, 2, 1, p(dx))
    np.testing.assert_allclose(dx, xt.grad.numpy(), rtol=1e-6, atol=1e-6)


def test_losses_match_torch(orc):
    rng = np.random.default_rng(4)
    # softmax CE (the reference CE op semantics)
    B, Cc = 37, 11
    lg = rng.standard_normal((B, Cc)).astype(np.float32) * 3
    lab = rng.integers(0, Cc, B).astype(np.int32)
    dx = np.zeros_like(lg)
    loss = orc.orc_softmax_ce(p(lg), B, Cc, p(lab), 1.0, 128.0, p(dx))
    lt = torch.from_numpy(lg).double().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(lt, torch.from_numpy(lab).long())
    ref.backward()
    assert abs(loss - ref.item()) < 1e-7 * abs(ref.item())  # probabilities stored as float (model.cpp:126)
    np.testing.assert_allclose(dx, 128 * lt.grad.numpy(), rtol=1e-5, atol=1e-6)
    # sigmoid BCE over labelled anchors
    n = 300
    x = rng.standard_normal(n).astype(np.float32) * 4
    t = rng.integers(-1, 2, n).astype(np.int8)
    g = np.zeros_like(x)
    valid = t >= 0
    loss = orc.orc_sigmoid_bce(p(x), p(t), n, float(valid.sum()), 4.0, p(g))
    xt = torch.from_numpy(x[valid]).double().requires_grad_(True)
    ref = torch.nn.functional.binary_cross_entropy_with_logits(xt, torch.from_numpy(t[valid]).double())
    ref.backward()
    assert abs(loss - ref.item()) < 1e-9
    np.testing.assert_allclose(g[valid], 4 * xt.grad.numpy(), rtol=1e-5, atol=1e-7)
    assert np.all(g[~valid] == 0)
    # smooth-L1
    rows = 50
    pr = rng.standard_normal((rows, 4)).astype(np.float32)
    tg = rng.standard_normal((rows, 4)).astype(np.float32)
    wt = (rng.random(rows) < 0.5).astype(np.float32)
    d = np.zeros_like(pr)
    loss = orc.orc_smooth_l1(p(pr), p(tg), p(wt), rows, 1 / 9, 256.0, 1.0, p(d))
    m = wt > 0
    pt = torch.from_numpy(pr[m]).double().requires_grad_(True)
    ref = torch.nn.functional.smooth_l1_loss(pt, torch.from_numpy(tg[m]).double(), beta=1 / 9, reduction="sum") / 256
    ref.backward()
    assert abs(loss - ref.item()) < 1e-9
    np.testing.assert_allclose(d[m], pt.grad.numpy(), rtol=1e-5, atol=1e-7)


def test_anchor_targets_known_answer(orc):
    # 4 anchors: exact match with GT -> fg; disjoint -> bg; half-overlap -> ignore;
    # one straddling the image -> ignore
    an = np.array([[10, 10, 50, 50], [200, 200, 240, 240], [30, 10, 70, 50], [-5, 0, 20, 20]], np.float32)
    gt = np.array([[10, 10, 50, 50]], np.float32)
    lab = np.zeros(4, np.int8)
    tg = np.zeros((4, 4), np.float32)
    orc.orc_anchor_targets(p(an), 4, p(gt), 1, 300.0, 300.0, 7, 0.7, 0.3, 256, 0.5, p(lab), p(tg))
    assert lab.tolist() == [1, 0, -1, -1]
    assert np.all(tg[0] == 0)  # exact match -> zero regression target
    # fg cap: 5 identical fg anchors, batch 4, fg_frac 0.5 -> 2 fg kept
    an5 = np.repeat(gt, 5, 0)
    lab5 = np.zeros(5, np.int8)
    tg5 = np.zeros((5, 4), np.float32)
    orc.orc_anchor_targets(p(an5), 5, p(gt), 1, 300.0, 300.0, 7, 0.7, 0.3, 4, 0.5, p(lab5), p(tg5))
    assert (lab5 == 1).sum() == 2 and (lab5 == -1).sum() == 3


def test_proposal_targets_known_answer(orc):
    props = np.array([[10, 10, 50, 50], [12, 10, 52, 50], [200, 200, 260, 260]], np.float32)
    gt = np.array([[10, 10, 50, 50]], np.float32)
    cls = np.array([7], np.int32)
    out = np.zeros((8, 4), np.float32)
    lab = np.zeros(8, np.int32)
    tg = np.zeros((8, 4), np.float32)
    src = np.zeros(8, np.int32)
    S = orc.orc_proposal_targets(p(props), 3, p(gt), p(cls), 1, 11, 0.5, 0.5, 0.0, 8, 0.25, p(out), p(lab), p(tg),
                                 p(src))
    # candidates: 3 proposals + the GT itself; fg = {0,1,3} capped at round(0.25*8)=2, bg = {2}
    assert S == 3
    assert (lab[:S] == 7).sum() == 2 and lab[2] == 0
    assert src[2] == 2
    assert list(src[:2]) == sorted(src[:2])  # fg in index order


def test_proposals_small_case(orc):
    # three anchors, zero deltas: proposals = clipped anchors in score order with NMS
    an = np.array([[0, 0, 10, 10], [1, 1, 11, 11], [20, 20, 30, 30]], np.float32)
    dl = np.zeros((3, 4), np.float32)
    sc = np.array([0.1, 0.9, 0.5], np.float32)
    rois = np.zeros((3, 4), np.float32)
    rs = np.zeros(3, np.float32)
    order = np.zeros(3, np.int32)
    n = orc.orc_proposals(p(sc), p(dl), p(an), 3, 100.0, 100.0, 3, 0.5, 3, p(rois), p(rs), p(order))
    assert list(order) == [1, 2, 0]
    assert n == 2  # anchor 0 suppressed by anchor 1 (IoU 81/119 > 0.5)
    assert rois.tolist()[:2] == [[1, 1, 11, 11], [20, 20, 30, 30]]
