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


@pytest.mark.parametrize("n_img,pre_k,post_k", [(2, 12000, 2000), (1, 2000, 300), (1, 50, 7), (1, 300, 2000), (2, 130, 129)])
def test_rpn_proposal_bit_exact(orc, n_img, pre_k, post_k):
    """BASELINE config C3: logits N(0,2), deltas N(0,0.2), 50x84x15 anchors, 12000 -> 2000 at IoU 0.7"""
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
