"""GPU parity of the detection operators (C ABI) against the CPU restatement:
anchors, the RPN proposal layer (bit-exact top-k order, NMS keep list and
boxes on BASELINE config C3 shapes), RoIAlign forward/backward (fp32 tight,
fp16 within 1e-2, backward bitwise deterministic), softmax-CE."""
import numpy as np
import pytest

import oracle
from oracle import p
from tests.util import assert_close

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

C3_SCALES = (32.0, 64.0, 128.0, 256.0, 512.0)
RATIOS = (0.5, 1.0, 2.0)


def test_anchors_bit_exact(orc):
    from paper_1903_05831_b200 import simdet as sd
    H, W = 50, 84
    a = sd.make_anchors(H, W, 16.0, C3_SCALES, RATIOS).cpu().numpy()
    ref = np.zeros_like(a)
    s, r = np.array(C3_SCALES, np.float32), np.array(RATIOS, np.float32)
    orc.orc_anchors(H, W, 16.0, p(s), 5, p(r), 3, p(ref))
    assert np.array_equal(a.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("n_img,pre_k,post_k", [(2, 12000, 2000), (1, 2000, 300), (1, 50, 7), (1, 300, 2000), (2, 130, 129),
                                                (2, 12000, 5000), (1, 4100, 4100), (1, 12000, 9000),
                                                (1, 8200, 8200)])
def test_rpn_proposal_bit_exact(orc, n_img, pre_k, post_k):
    """BASELINE config C3: logits N(0,2), deltas N(0,0.2), 50x84x15 anchors, 12000 -> 2000 at IoU 0.7.
    The NMS mask is computed in bands of 4096 candidates, the scan resuming band
    by band until post_k boxes are kept: (12000, 5000) and (4100, 4100) need a
    second band, (12000, 9000) and (8200, 8200) all three (the last one a
    single word wide)."""
    from paper_1903_05831_b200 import simdet as sd
    H, W, A, Ap = 50, 84, 15, 16
    rng = np.random.default_rng(pre_k + n_img)
    lg = (rng.standard_normal((n_img, H * W, Ap)) * 2).astype(np.float16)
    dl = (rng.standard_normal((n_img, H * W, 4 * Ap)) * 0.2).astype(np.float16)
    lg[:, :5, 0] = lg[:, 5:10, 0]  # exact score ties (index order must break them)
    anchors = sd.make_anchors(H, W, 16.0, C3_SCALES, RATIOS)
    rois, scores, count, order = sd.rpn_proposal(torch.from_numpy(lg).cuda(), torch.from_numpy(dl).cuda(), anchors, A,
                                                 pre_k, 0.7, post_k, 800.0, 1333.0)
    torch.cuda.synchronize()
    an = anchors.cpu().numpy()
    for j in range(n_img):
        l = np.ascontiguousarray(lg[j, :, :A].astype(np.float32).reshape(-1))
        d = np.ascontiguousarray(dl[j].astype(np.float32)[:, : 4 * A].reshape(-1))
        rr = np.zeros((post_k, 4), np.float32)
        rs = np.zeros(post_k, np.float32)
        k = min(pre_k, H * W * A)
        oo = np.zeros(k, np.int32)
        n = orc.orc_proposals(p(l), p(d), p(an), H * W * A, 800.0, 1333.0, pre_k, 0.7, post_k, p(rr), p(rs), p(oo))
        assert np.array_equal(order[j].cpu().numpy(), oo), "top-k order"
        assert int(count[j]) == n
        assert np.array_equal(rois[j, :n].cpu().numpy().view(np.uint32), rr[:n].view(np.uint32)), "NMS boxes"
        assert np.array_equal(scores[j, :n].cpu().numpy(), rs[:n])


def _rois(rng, R, N, H, W):
    b = rng.integers(0, N, R)
    x1 = rng.uniform(-40, W * 16, R)
    y1 = rng.uniform(-40, H * 16, R)
    return np.stack([b, x1, y1, x1 + rng.uniform(1, 400, R), y1 + rng.uniform(1, 300, R)], 1).astype(np.float32)


@pytest.mark.parametrize("fp16", [False, True])
@pytest.mark.parametrize("P", [7, 14])
def test_roialign_fwd_bwd(orc, fp16, P):
    from paper_1903_05831_b200 import simdet as sd
    rng = np.random.default_rng(P + fp16)
    N, Cc, H, W, R = 2, 64, 50, 84, 300
    feat = rng.standard_normal((N, Cc, H, W)).astype(np.float32)
    if fp16:
        feat = feat.astype(np.float16).astype(np.float32)
    rois = _rois(rng, R, N, H, W)
    out_ref = np.zeros((R, Cc, P, P), np.float32)
    orc.orc_roialign_fwd(p(feat), N, Cc, H, W, p(rois), R, P, 1 / 16, 2, 1, p(out_ref))
    dy = rng.standard_normal(out_ref.shape).astype(np.float32)
    if fp16:
        dy = dy.astype(np.float16).astype(np.float32)
    dx_ref = np.zeros_like(feat)
    orc.orc_roialign_bwd(p(dy), N, Cc, H, W, p(rois), R, P, 1 / 16, 2, 1, p(dx_ref))
    tdt = torch.float16 if fp16 else torch.float32
    rt = torch.from_numpy(rois).cuda()
    out = sd.roialign_forward(torch.from_numpy(feat).to("cuda", tdt), rt, P, 1 / 16, 2)
    dx = sd.roialign_backward(torch.from_numpy(dy).to("cuda", tdt), (N, Cc, H, W), rt, P, 1 / 16, 2)
    dx2 = sd.roialign_backward(torch.from_numpy(dy).to("cuda", tdt), (N, Cc, H, W), rt, P, 1 / 16, 2)
    torch.cuda.synchronize()
    tol = 1e-2 if fp16 else 1e-5
    assert_close(out, out_ref, tol, "roialign fwd")
    assert_close(dx, dx_ref, tol, "roialign bwd")
    assert torch.equal(dx, dx2), "backward must be bitwise deterministic"


def test_softmax_ce_matches_reference_op(orc):
    from paper_1903_05831_b200 import simdet as sd
    rng = np.random.default_rng(9)
    R, ncls = 1024, 81
    lg = (rng.standard_normal((R, ncls)) * 3).astype(np.float32)
    lab = rng.integers(0, ncls, R).astype(np.int32)
    dx_ref = np.zeros_like(lg)
    loss_ref = orc.orc_softmax_ce(p(lg), R, ncls, p(lab), 1.0, 128.0, p(dx_ref))
    scale = torch.tensor([128.0], dtype=torch.float64, device="cuda")
    loss, dx = sd.softmax_ce(torch.from_numpy(lg).cuda(), torch.from_numpy(lab).cuda(), scale)
    torch.cuda.synchronize()
    assert abs(loss.item() - loss_ref) <= 1e-9 * abs(loss_ref)
    assert_close(dx, dx_ref, 1e-6, "dlogits")


def _gt_boxes(rng, G, img_h, img_w, wh=(8.0, 512.0)):
    cx, cy = rng.uniform(0, img_w, G), rng.uniform(0, img_h, G)
    w = np.exp(rng.uniform(np.log(wh[0]), np.log(wh[1]), G))
    h = np.exp(rng.uniform(np.log(wh[0]), np.log(wh[1]), G))
    return np.stack([np.clip(cx - w / 2, 0, img_w), np.clip(cy - h / 2, 0, img_h), np.clip(cx + w / 2, 0, img_w),
                     np.clip(cy + h / 2, 0, img_h)], 1).astype(np.float32)


@pytest.mark.parametrize("counts", [(7, 12), (0, 1), (32, 3)])
def test_anchor_targets_abi_bit_exact(orc, counts):
    """sdb_anchor_targets at the C4 anchor grid (50x84x15) vs orc_anchor_targets:
    labels bit-exact (incl. the keyed fg/bg subsampling), targets to 1e-6"""
    from paper_1903_05831_b200 import simdet as sd
    H, W, img_h, img_w, Gs = 50, 84, 800.0, 1333.0, 32
    rng = np.random.default_rng(sum(counts))
    anchors = sd.make_anchors(H, W, 16.0, C3_SCALES, RATIOS)
    an = anchors.cpu().numpy()
    nA = an.shape[0]
    gt = np.zeros((2, Gs, 4), np.float32)
    for j, c in enumerate(counts):
        gt[j, :c] = _gt_boxes(rng, c, img_h, img_w)
    cnt = np.array(counts, np.int32)
    keys = np.array([orc.orc_mix64(0xA11C0000, 11 + j) for j in range(2)], np.uint64)
    lab, tg = sd.anchor_targets(anchors, torch.from_numpy(gt).cuda(), torch.from_numpy(cnt).cuda(),
                                torch.from_numpy(keys.view(np.int64)).cuda(), img_h, img_w)
    torch.cuda.synchronize()
    for j, c in enumerate(counts):
        rl = np.zeros(nA, np.int8)
        rt = np.zeros((nA, 4), np.float32)
        orc.orc_anchor_targets(p(an), nA, p(np.ascontiguousarray(gt[j, :c])), c, img_h, img_w, int(keys[j]), 0.7, 0.3,
                               256, 0.5, p(rl), p(rt))
        assert np.array_equal(lab[j].cpu().numpy(), rl), f"labels img {j}"
        np.testing.assert_allclose(tg[j].cpu().numpy(), rt, rtol=1e-6, atol=1e-6)
        if c == 0:
            assert (rl == 1).sum() == 0


def test_proposal_targets_abi_bit_exact(orc):
    """sdb_proposal_targets at C4 sizes (2000 proposals + GT, 512 RoIs at 1:3) vs
    orc_proposal_targets: sampled boxes and labels bit-exact, targets to 1e-5"""
    from paper_1903_05831_b200 import simdet as sd
    rng = np.random.default_rng(21)
    n_img, Pst, Gs, img_h, img_w = 2, 2000, 32, 800.0, 1333.0
    props = np.zeros((n_img, Pst, 4), np.float32)
    pc = np.array([2000, 1377], np.int32)
    gt = np.zeros((n_img, Gs, 4), np.float32)
    gcls = np.zeros((n_img, Gs), np.int32)
    gcnt = np.array([7, 19], np.int32)
    for j in range(n_img):
        g = _gt_boxes(rng, gcnt[j], img_h, img_w)
        gt[j, :gcnt[j]] = g
        gcls[j, :gcnt[j]] = rng.integers(1, 81, gcnt[j])
        # proposals: jittered GT copies (foreground) and random boxes (background)
        k = pc[j]
        src = g[rng.integers(0, gcnt[j], k)]
        jit = rng.normal(0, 12, (k, 4)).astype(np.float32)
        rnd = _gt_boxes(rng, k, img_h, img_w)
        pick = rng.random(k) < 0.3
        props[j, :k] = np.where(pick[:, None], np.clip(src + jit, 0, [img_w, img_h, img_w, img_h]), rnd)
    keys = np.array([orc.orc_mix64(0x5A3B0000, 5 + j) for j in range(n_img)], np.uint64)
    T = lambda a: torch.from_numpy(a).cuda()
    rois, labels, targets, count = sd.proposal_targets(T(props), T(pc), T(gt), T(gcls), T(gcnt),
                                                       T(keys.view(np.int64)), batch=512, fg_frac=0.25)
    torch.cuda.synchronize()
    for j in range(n_img):
        orr = np.zeros((512, 4), np.float32)
        ol = np.zeros(512, np.int32)
        ot = np.zeros((512, 4), np.float32)
        S = orc.orc_proposal_targets(p(np.ascontiguousarray(props[j, :pc[j]])), int(pc[j]),
                                     p(np.ascontiguousarray(gt[j, :gcnt[j]])), p(np.ascontiguousarray(gcls[j, :gcnt[j]])),
                                     int(gcnt[j]), int(keys[j]), 0.5, 0.5, 0.0, 512, 0.25, p(orr), p(ol), p(ot), None)
        assert int(count[j]) == S
        gr = rois[j * 512:(j + 1) * 512].cpu().numpy()
        gl = labels[j * 512:(j + 1) * 512].cpu().numpy()
        assert np.all(gr[:S, 0] == j)
        assert np.array_equal(gr[:S, 1:].view(np.uint32), orr[:S].view(np.uint32))
        assert np.array_equal(gl[:S], ol[:S]) and (gl[:S] > 0).sum() > 0
        assert np.all(gl[S:] == -1)
        np.testing.assert_allclose(targets[j * 512:j * 512 + S].cpu().numpy(), ot[:S], rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("fp16", [False, True])
def test_detection_losses_abi(orc, fp16):
    """sdb_rpn_bce / sdb_rpn_smoothl1 / sdb_smoothl1 vs the restated losses
    (orc_sigmoid_bce, orc_smooth_l1): loss to 1e-9 relative (fp32 inputs) and
    gradients (scaled by the loss scale) to 1e-6 / fp16 rounding"""
    from paper_1903_05831_b200 import simdet as sd
    rng = np.random.default_rng(31 + fp16)
    tdt = torch.float16 if fp16 else torch.float32
    ndt = np.float16 if fp16 else np.float32
    n_loc, A, Ap = 50 * 84, 15, 16
    lg = (rng.standard_normal((n_loc, Ap)) * 2).astype(ndt)
    lab = rng.choice(np.array([-1, 0, 1], np.int8), n_loc * A, p=[0.95, 0.04, 0.01])
    scale = torch.tensor([128.0], dtype=torch.float64, device="cuda")
    loss, dlg = sd.rpn_bce(torch.from_numpy(lg).cuda(), torch.from_numpy(lab).cuda(), A, scale)
    x = np.ascontiguousarray(lg[:, :A].astype(np.float32).reshape(-1))
    dref = np.zeros_like(x)
    norm = float((lab >= 0).sum())
    lref = orc.orc_sigmoid_bce(p(x), p(lab), x.size, norm, 128.0, p(dref))
    assert abs(loss.item() - lref) <= 1e-9 * abs(lref)
    assert_close(dlg[:, :A].float().reshape(-1), dref, 1e-3 if fp16 else 1e-6, "rpn bce grad")
    assert torch.all(dlg[:, A:] == 0)
    # RPN smooth-L1, beta 1/9, normalised by 256 x images
    dl = (rng.standard_normal((n_loc, 4 * Ap)) * 0.2).astype(ndt)
    tg = (rng.standard_normal((n_loc * A, 4)) * 0.3).astype(np.float32)
    loss, ddl = sd.rpn_smoothl1(torch.from_numpy(dl).cuda(), torch.from_numpy(lab).cuda(), torch.from_numpy(tg).cuda(),
                                A, 1.0 / 9.0, 512.0, scale)
    pr = np.ascontiguousarray(dl[:, :4 * A].astype(np.float32).reshape(-1, 4))
    wt = (lab == 1).astype(np.float32)
    dref = np.zeros_like(pr)
    lref = orc.orc_smooth_l1(p(pr), p(tg), p(wt), pr.shape[0], 1.0 / 9.0, 512.0, 128.0, p(dref))
    assert abs(loss.item() - lref) <= 1e-9 * abs(lref)
    assert_close(ddl[:, :4 * A].float().reshape(-1, 4), dref, 1e-3 if fp16 else 1e-6, "rpn smooth-l1 grad")
    # RCNN class-specific smooth-L1 (beta 1), / #RoIs with label >= 0
    R, ncls = 1024, 81
    ld = 4 * ncls + 4
    pred = (rng.standard_normal((R, ld)) * 0.5).astype(ndt)
    rl = rng.integers(0, ncls, R).astype(np.int32)
    rl[rng.random(R) < 0.6] = 0
    rl[-7:] = -1
    rt = (rng.standard_normal((R, 4)) * 0.5).astype(np.float32)
    loss, dpr = sd.smoothl1(torch.from_numpy(pred).cuda(), torch.from_numpy(rl).cuda(), torch.from_numpy(rt).cuda(), 1.0,
                            scale)
    sel = np.stack([pred[i, 4 * max(rl[i], 0): 4 * max(rl[i], 0) + 4].astype(np.float32) for i in range(R)])
    wt = (rl > 0).astype(np.float32)
    dref = np.zeros_like(sel)
    lref = orc.orc_smooth_l1(p(sel), p(rt), p(wt), R, 1.0, float((rl >= 0).sum()), 128.0, p(dref))
    assert abs(loss.item() - lref) <= 1e-9 * abs(lref)
    dg = dpr.float().cpu().numpy()
    dsel = np.stack([dg[i, 4 * max(rl[i], 0): 4 * max(rl[i], 0) + 4] for i in range(R)])
    assert_close(dsel, dref, 1e-3 if fp16 else 1e-6, "rcnn smooth-l1 grad")
    mask = np.ones_like(dg, bool)
    for i in range(R):
        if rl[i] > 0:
            mask[i, 4 * rl[i]: 4 * rl[i] + 4] = False
    assert np.all(dg[mask] == 0)


@pytest.mark.parametrize("fp16", [True, False])
def test_roialign_c3_shape(orc, fp16):
    """BASELINE config C3 shape: 8 x 1024-channel 50x84 features, 8 x 512 RoIs,
    RoIAlign 14x14 (sampling ratio 2) forward and backward.  RoIAlign is
    channel-separable, so the CPU restatement runs on a 64-channel subset (both
    ends of the channel range: first and last slab of every kernel tiling)."""
    from paper_1903_05831_b200 import simdet as sd
    rng = np.random.default_rng(41 + fp16)
    N, Cc, H, W, P = 8, 1024, 50, 84, 14
    R = N * 512
    tdt = torch.float16 if fp16 else torch.float32
    feat = torch.randn((N, Cc, H, W), device="cuda").to(tdt)
    rois = _rois(rng, R, N, H, W)
    rois[:, 0] = np.repeat(np.arange(N), 512)
    rt = torch.from_numpy(rois).cuda()
    dy = torch.randn((R, Cc, P, P), device="cuda").to(tdt)
    out = sd.roialign_forward(feat, rt, P, 1 / 16, 2)
    dx = sd.roialign_backward(dy, (N, Cc, H, W), rt, P, 1 / 16, 2)
    dx2 = sd.roialign_backward(dy, (N, Cc, H, W), rt, P, 1 / 16, 2)
    torch.cuda.synchronize()
    assert torch.equal(dx, dx2), "backward must be bitwise deterministic"
    ch = np.r_[0:32, Cc - 32:Cc]
    f_sub = np.ascontiguousarray(feat[:, ch].float().cpu().numpy())
    dy_sub = np.ascontiguousarray(dy[:, ch].float().cpu().numpy())
    out_ref = np.zeros((R, len(ch), P, P), np.float32)
    orc.orc_roialign_fwd(p(f_sub), N, len(ch), H, W, p(rois), R, P, 1 / 16, 2, 1, p(out_ref))
    dx_ref = np.zeros_like(f_sub)
    orc.orc_roialign_bwd(p(dy_sub), N, len(ch), H, W, p(rois), R, P, 1 / 16, 2, 1, p(dx_ref))
    tol = 1e-2 if fp16 else 1e-5
    assert_close(out[:, ch], out_ref, tol, "roialign fwd C3")
    assert_close(dx[:, ch], dx_ref, tol, "roialign bwd C3")
